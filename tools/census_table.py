"""Prints profiles/r4_census.txt from paper_1901_04200_b200/census.py."""
import os
import sys

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
from paper_1901_04200_b200 import census  # noqa: E402

print("""# r4 census: floating-point instructions per path of the pass kernels (ncu, --clock-control none)
# executed = thread-level DADD+DMUL+DFMA (fp32 mode: FADD+FMUL+FFMA), predicate on, / paths of the launch
# algorithmic = executed - redundant (the central branch on tail slots + padding slots; census.py)
# sources (one tools/gpu_profile.sh r4 session, read by tools/census_from_ncu.py): r4_cfg3_z{0,1}_raw.csv.gz (fp64, 2^20 paths,
#          --set full), r4_census_{cfg1,cfg2,cfg4}_fp64_*.csv, r4_census_{cfg1,cfg2}_fp32_*.csv, r4_cfg3f32_z{0,1}_raw.csv.gz;
#          z0 = LTG_ZSTORE=0 (pass 2 regenerates its draws), z1 = default (every chunk's draws stored at these sizes)
""")
print(f"{'config':16s} {'prec':5s} {'kernel':12s} {'executed':>10s} {'redundant':>10s} {'algorithmic':>12s}")
for (name, prec), d in census.EXECUTED.items():
    for k, v in d.items():
        print(f"{name:16s} {prec:5s} {k:12s} {v:10.1f} {census.redundant(name, prec, k):10.1f} "
              f"{census.algorithmic(name, prec, k):12.1f}")
print("\n# DRAM bytes per path (dram__bytes_read + write), cfg3 at 2^20:")
for (name, prec), d in census.DRAM.items():
    print(f"{name:16s} {prec:5s} " + "  ".join(f"{k} {v:.1f}" for k, v in d.items()))
print("""
# kernel times at 2^20 paths (ncu gpu__time_duration, serialised, cold):
#   fp64 pass 1  9.68 ms (z0) /  9.93 ms (z1, writes the draw store); pass 2  9.91 ms (z0) / 3.80 ms (z1)
#   fp32 pass 1  4.33 ms (z0) /  4.54 ms (z1);                        pass 2  4.96 ms (z0) / 2.15 ms (z1)
# pipe use (cfg3 fp64, z0): pass 1 FP64 pipe 64.8%, issue 64.7%; pass 2 FP64 pipe 64.0%, issue 65.6%
#            (fp32, z0):   pass 1 issue 75.7%; pass 2 issue 77.3%
# warp instructions per path-step (fp64, z0): pass 1 289 (r3: 308, r2: 324), pass 2 300 (r3: 315, r2: 339);
#            (fp32, z0):   pass 1 151 (r3: 175), pass 2 177 (r3: 200)""")
