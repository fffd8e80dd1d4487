"""Frozen FP64 work census of the ∇G kernels (the roofline numerator).

W = FP64 instructions per path that the algorithm executes for useful lanes:
thread-level DADD + DMUL + DFMA with predicate on, counted by ncu
(smsp__sass_thread_inst_executed_op_{dadd,dmul,dfma}_pred_on.sum) on one
launch and divided by the launch's path count. Lanes idled by divergence
are NOT counted, so achieved/peak is the useful fraction of the FP64 pipe.
Numbers are frozen per (config, precision, kernel) in DESIGN.md §5 and only
change when the algorithm changes (not when it is tuned).

cfg3/cfg5 are frozen from the first implementation (profiles/r1_v1_cfg3_full.txt),
which evaluated exactly one AS241 branch per draw. cfg1/cfg2/cfg4 were first
counted on the v4 kernels (profiles/r1_v4_census.txt), which evaluate the
central branch on every draw (about 6 FP64 instructions of redundant work per
tail draw, ~2% of the total) — those fractions are slightly flattering.
"""
from __future__ import annotations

# per-path thread-level FP64 instruction counts
PASS1_FP64 = {"cfg3_heston:fp64": 107979.0, "cfg1_gbm:fp64": 2394.0,
              "cfg2_localvol:fp64": 9945.0, "cfg4_basket16:fp64": 67307.0}
PASS2_FP64 = {"cfg3_heston:fp64": 143004.0, "cfg1_gbm:fp64": 2960.0,
              "cfg2_localvol:fp64": 12346.0, "cfg4_basket16:fp64": 503.0}
# fp32 mode: thread-level FADD + FFMA + FMUL per path (the arithmetic the FP32
# pipe executes), counted without the draw store on the r1 kernels (cfg3 fp32
# at 2^18, LTG_ZSTORE=0); the mode also keeps ~6-7k FP64 instructions per pass
# (the exact uniform and tail arguments) and all of Philox
PASS1_FP32 = {"cfg3_heston:fp32": 45249.3}
PASS2_FP32 = {"cfg3_heston:fp32": 67958.8}
# per-path DRAM bytes (ncu dram__bytes_read+write / paths), latest capture without the
# draw store (profiles/r1_v12_cfg3_noz_full.txt: the regime of cfg5 on one GPU)
PASS1_DRAM = {"cfg3_heston:fp64": 1455.8}
PASS2_DRAM = {"cfg3_heston:fp64": 1526.4}


def _key(name: str, precision: str):
    base = "cfg3_heston" if name.startswith("cfg5") else name
    return f"{base}:{precision}"


def pass1_fp64_per_path(name: str, precision: str = "fp64"):
    return PASS1_FP64.get(_key(name, precision))


def pass2_fp64_per_path(name: str, precision: str = "fp64"):
    return PASS2_FP64.get(_key(name, precision))


def dram_bytes_per_path(name: str, precision: str = "fp64", kernel: str = "pass2"):
    table = PASS1_DRAM if kernel == "pass1" else PASS2_DRAM
    return table.get(_key(name, precision))


def pass1_fp32_per_path(name: str, precision: str = "fp32"):
    return PASS1_FP32.get(_key(name, precision))


def pass2_fp32_per_path(name: str, precision: str = "fp32"):
    return PASS2_FP32.get(_key(name, precision))
