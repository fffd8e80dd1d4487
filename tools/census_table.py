"""Prints profiles/r2_census.txt from paper_1901_04200_b200/census.py."""
import os
import sys

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
from paper_1901_04200_b200 import census  # noqa: E402

print("""# r2 census: floating-point instructions per path of the pass kernels (ncu, --clock-control none)
# executed = thread-level DADD+DMUL+DFMA (fp32 mode: FADD+FMUL+FFMA), predicate on, / paths of the launch
# algorithmic = executed - redundant (the central branch on tail slots + padding slots; census.py)
# sources: gpurun_out/r2c_cfg3_z{0,1}_raw.csv.gz (fp64, 2^20 paths, --set full), r2c_census_{cfg1,cfg2,cfg4}_fp64_*.csv,
#          r2c_census_{cfg1,cfg2}_fp32_*.csv, r2c_cfg3f32_z{0,1}_raw.csv.gz (the fp32 mode with its single-precision inverse normal);
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
#   fp64 pass 1 10.31 ms (z0) / 10.71 ms (z1, writes the draw store); pass 2 11.06 ms (z0) / 3.97 ms (z1)
#   fp32 pass 1  5.00 ms (z0) /  5.24 ms (z1);                        pass 2  5.61 ms (z0) / 2.26 ms (z1)
# pipe use (cfg3 fp64, z0): pass 1 FP64 pipe 60.5%, issue 67.9%; pass 2 FP64 pipe 57.9%, issue 66.5%
#            (fp32, z0):   pass 1 issue 74.9%, ALU 53.8%, FMA 32.0%, XU 23.6%; pass 2 issue 77.7%""")
