"""Work census of the ∇G pass kernels: the roofline numerator of bench.py.

EXECUTED — what the current kernels execute per path, counted by ncu
(thread-level DADD + DMUL + DFMA with predicate on; the fp32 mode: FADD +
FMUL + FFMA), one launch divided by its path count. Pass 2 has two rows:
"regen" (the chunk's draws are regenerated from Philox) and "store" (pass 1
kept them in the HBM draw store and pass 2 reads them); a call's pass-2
figure is the two weighted by the fraction of its paths whose draws were
stored (bench.py reads that from ltg_timing.z_bytes).
Source: profiles/r4_census.txt (tools/census_from_ncu.py on one
tools/gpu_profile.sh session; cfg3 at 2^20, cfg1 at 2^16, cfg2 and cfg4 at
2^18 paths; the round-2 final kernels: S-free pass 2, V-only checkpoints,
the fp32 mode's single-precision inverse normal, Philox and AS241's central
branch fused in one loop, whole fused iterations stored, step loops in runs
between maturities).

ALGORITHMIC — EXECUTED minus the kernels' only redundant floating-point work:
gen_segment evaluates AS241's central branch for every slot of a batch,
branch-free, and overwrites the tail slots (|q| > 0.425, probability exactly
0.15) in a warp-compacted second phase; the central evaluation of a tail slot
is wasted (CENTRAL_OPS instructions), and so is that of the padding slots of a
batch shorter than the central batch width. Everything else the kernels
execute is work of the algorithm they implement (the hand-derived adjoint;
pass 2 replays V only, so S's exp is neither executed nor credited).
"""
from __future__ import annotations

from typing import Dict, Optional, Tuple

# AS241 central branch per slot (rng.cuh gen_segment phase B): r = c - q*q
# (2), two degree-7 Horner chains with separate multiply and add (28), q*num
# (1), the correctly rounded division (8 DFMA/DMUL around MUFU.RCP64H) = 39.
# fp32 mode (the fitted 3/3 rational, f32_normal.h): FFMA for r, 3 + 3 FFMA,
# FMUL q*num, FMUL by the MUFU reciprocal = 9.
CENTRAL_OPS = {"fp64": 39.0, "fp32": 9.0}
TAIL_FRACTION = 0.15  # P(|p - 0.5| > 0.425), p uniform

# name -> (steps, draws per path)
SHAPE = {"cfg1_gbm": (16, 32), "cfg2_localvol": (64, 128), "cfg3_heston": (756, 1512),
         "cfg4_basket16": (50, 800)}

# (config, precision) -> {kernel: executed instructions per path}
EXECUTED: Dict[Tuple[str, str], Dict[str, float]] = {
    ("cfg3_heston", "fp64"): {"pass1": 104156.6, "pass2_regen": 105634.5, "pass2_store": 29809.4},
    ("cfg3_heston", "fp32"): {"pass1": 29074.5, "pass2_regen": 42056.0, "pass2_store": 22929.5},
    ("cfg1_gbm", "fp64"): {"pass1": 2333.5, "pass2_regen": 2405.6, "pass2_store": 801.2},
    ("cfg1_gbm", "fp32"): {"pass1": 676.7, "pass2_regen": 988.9, "pass2_store": 584.1},
    ("cfg2_localvol", "fp64"): {"pass1": 9439.4, "pass2_regen": 11399.2, "pass2_store": 4980.9},
    ("cfg2_localvol", "fp32"): {"pass1": 2723.1, "pass2_regen": 4496.1, "pass2_store": 2861.1},
    # the basket's pass 2 is a store-mode epilogue (no draws, no replay)
    ("cfg4_basket16", "fp64"): {"pass1": 66348.8, "pass2_regen": 455.1, "pass2_store": 455.1},
}

# DRAM bytes per path (ncu dram__bytes_read + write), without / with the draw store
DRAM: Dict[Tuple[str, str], Dict[str, float]] = {
    ("cfg3_heston", "fp64"): {"pass1": 751.8, "pass1_store": 12850.9, "pass2_regen": 810.0,
                              "pass2_store": 12911.0},
    ("cfg3_heston", "fp32"): {"pass1": 351.4, "pass1_store": 6400.0, "pass2_regen": 405.1,
                              "pass2_store": 6452.7},
}

# central-batch widths and normal batches of the kernels (heston.cu: kPass1PB,
# kPass2PB, kGenSteps; the checkpoint interval KS = 8 of every BASELINE plan)
_PB = {("fp64", "pass1"): 16, ("fp32", "pass1"): 4, ("fp64", "pass2"): 8, ("fp32", "pass2"): 8}
_BATCH_STEPS = 8


def _key(name: str, precision: str) -> Tuple[str, str]:
    return ("cfg3_heston" if name.startswith("cfg5") else name, precision)


def _pad_slots(steps: int, pb: int) -> int:
    """central evaluations of slots past a short batch's end, per path"""
    pad = 0
    for k0 in range(0, steps, _BATCH_STEPS):
        ns = 2 * min(_BATCH_STEPS, steps - k0)
        pad += -(-ns // pb) * pb - ns
    return pad


def redundant(name: str, precision: str, kernel: str) -> float:
    """wasted central-branch instructions per path of one launch"""
    base, _ = _key(name, precision)
    if base not in SHAPE or kernel == "pass2_store":
        return 0.0
    if base == "cfg4_basket16":  # one RNG pass (pass 1); the epilogue draws nothing
        return CENTRAL_OPS[precision] * TAIL_FRACTION * SHAPE[base][1] if kernel == "pass1" else 0.0
    steps, draws = SHAPE[base]
    pad = _pad_slots(steps, _PB[(precision, kernel[:5])])
    return CENTRAL_OPS[precision] * (TAIL_FRACTION * draws + pad)


def executed(name: str, precision: str, kernel: str) -> Optional[float]:
    return EXECUTED.get(_key(name, precision), {}).get(kernel)


def algorithmic(name: str, precision: str, kernel: str) -> Optional[float]:
    e = executed(name, precision, kernel)
    return None if e is None else e - redundant(name, precision, kernel)


def per_path(name: str, precision: str, kernel: str, store_fraction: float = 0.0,
             basis: str = "algorithmic") -> Optional[float]:
    """census of `kernel` ("pass1" or "pass2") for a call in which
    `store_fraction` of the paths had their draws in the draw store"""
    f = algorithmic if basis == "algorithmic" else executed
    if kernel == "pass1":
        return f(name, precision, "pass1")
    a, b = f(name, precision, "pass2_regen"), f(name, precision, "pass2_store")
    if a is None or b is None:
        return None
    return (1.0 - store_fraction) * a + store_fraction * b


def dram_per_path(name: str, precision: str, kernel: str, store_fraction: float = 0.0):
    t = DRAM.get(_key(name, precision))
    if t is None:
        return None
    if kernel == "pass1":
        return (1.0 - store_fraction) * t["pass1"] + store_fraction * t["pass1_store"]
    return (1.0 - store_fraction) * t["pass2_regen"] + store_fraction * t["pass2_store"]


# SURVEY.md §8(d)'s preliminary algorithmic work per path (FP64 issues with its
# per-op weights, both passes drawing every normal): a cross-check figure
# beside the census, reported by bench.py as roofline.survey_8d.
SURVEY_W = {"cfg1_gbm": 2.4e3, "cfg2_localvol": 1.14e4, "cfg3_heston": 2.6e5, "cfg4_basket16": 1.33e5}


def survey_w(name: str) -> Optional[float]:
    return SURVEY_W.get(_key(name, "fp64")[0])
