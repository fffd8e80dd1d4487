"""Frozen FP64 work census of the ∇G kernels (the roofline numerator).

W = FP64 instructions per path that the algorithm executes for useful lanes:
thread-level DADD + DMUL + DFMA with predicate on, counted by ncu
(smsp__sass_thread_inst_executed_op_{dadd,dmul,dfma}_pred_on.sum) on one
launch and divided by the launch's path count. Lanes idled by divergence
are NOT counted, so achieved/peak is the useful fraction of the FP64 pipe.
Numbers are frozen per (config, precision, kernel) in DESIGN.md §5 and only
change when the algorithm changes (not when it is tuned).
"""
from __future__ import annotations

from .kernels_meta import SEG_STEPS

# per-path thread-level FP64 instruction counts (ncu, profiles/)
# frozen from the first (v1) implementation, which evaluates exactly one
# polynomial per draw and log/sqrt only on tail lanes (profiles/r1_v1_cfg3_full.txt)
PASS2_FP64 = {"cfg3_heston:fp64": 143004.0}
PASS1_FP64 = {"cfg3_heston:fp64": 107979.0}
# per-path DRAM bytes of pass 2 (ncu dram__bytes_read+write / paths), latest capture
PASS2_DRAM = {"cfg3_heston:fp64": 780.8}


def _key(name: str, precision: str):
    base = "cfg3_heston" if name.startswith("cfg5") else name
    return f"{base}:{precision}"


def pass2_fp64_per_path(name: str, precision: str = "fp64"):
    return PASS2_FP64.get(_key(name, precision))


def pass1_fp64_per_path(name: str, precision: str = "fp64"):
    return PASS1_FP64.get(_key(name, precision))


def pass2_dram_bytes_per_path(name: str, precision: str = "fp64"):
    return PASS2_DRAM.get(_key(name, precision))


def ckpt_bytes(cfg) -> float:
    """HBM checkpoint table written by pass 1 and read by pass 2."""
    spec = cfg.spec
    if not hasattr(spec, "mc"):
        return 0.0
    nseg = (spec.mc.steps + SEG_STEPS - 1) // SEG_STEPS
    return float(max(0, nseg - 1)) * cfg.paths * 16
