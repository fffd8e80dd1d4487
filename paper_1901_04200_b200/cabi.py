"""ctypes mirror of include/lanetape_b200.h (structs and model marshalling).

Used by the Python-side binding of the CUDA engine (engine.py) and, as plain
type definitions, by the test-only oracle bindings.
"""
from __future__ import annotations

import ctypes as C
from typing import List, Sequence

from .model import BasketSpec, ModelSpec, CALL, PUT

LTG_OK, LTG_EINVAL, LTG_ENUMERIC, LTG_ECUDA = 0, 1, 2, 3


class HestonModelC(C.Structure):
    _fields_ = [
        ("mu", C.c_double), ("s0", C.c_double),
        ("kappa", C.c_double), ("theta", C.c_double), ("xi", C.c_double),
        ("rho", C.c_double), ("v0", C.c_double),
        ("t_nodes", C.POINTER(C.c_double)), ("n_t_nodes", C.c_uint32),
        ("s_nodes", C.POINTER(C.c_double)), ("n_s_nodes", C.c_uint32),
        ("leverage", C.POINTER(C.c_double)),
        ("inst_kind", C.POINTER(C.c_int32)),
        ("inst_strike", C.POINTER(C.c_double)),
        ("inst_maturity_step", C.POINTER(C.c_uint32)),
        ("n_instruments", C.c_uint32),
        ("steps", C.c_uint32),
        ("dt", C.c_double),
    ]


class BasketModelC(C.Structure):
    _fields_ = [
        ("n_assets", C.c_uint32),
        ("s0", C.POINTER(C.c_double)),
        ("r", C.c_double),
        ("chol", C.POINTER(C.c_double)),
        ("sigma", C.POINTER(C.c_double)),
        ("inst_asset", C.POINTER(C.c_uint32)),
        ("inst_kind", C.POINTER(C.c_int32)),
        ("inst_strike", C.POINTER(C.c_double)),
        ("inst_maturity_step", C.POINTER(C.c_uint32)),
        ("n_instruments", C.c_uint32),
        ("steps", C.c_uint32),
        ("dt", C.c_double),
    ]


class MCConfigC(C.Structure):
    _fields_ = [
        ("paths", C.c_uint64), ("seed", C.c_uint64),
        ("antithetic", C.c_int32), ("fresh_step2_paths", C.c_int32),
        ("memory_mode", C.c_int32), ("precision", C.c_int32),
    ]


class DrawsC(C.Structure):
    """ltg_draws: caller draws, path-major rows of dim doubles"""
    _fields_ = [("data", C.POINTER(C.c_double)), ("rows", C.c_uint64), ("dim", C.c_uint64)]


class ReportC(C.Structure):
    _fields_ = [
        ("G", C.c_double),
        ("means", C.POINTER(C.c_double)), ("lambda_", C.POINTER(C.c_double)),
        ("grad", C.POINTER(C.c_double)), ("std_errors", C.POINTER(C.c_double)),
        ("paths", C.c_uint64), ("seed", C.c_uint64), ("mode", C.c_int32),
    ]


class TimingC(C.Structure):
    _fields_ = [
        ("pass1_ms", C.c_double), ("pass2_ms", C.c_double), ("reduce_ms", C.c_double),
        ("total_ms", C.c_double), ("paths_pass1", C.c_uint64), ("paths_pass2", C.c_uint64),
        ("launches", C.c_uint32), ("seg_steps", C.c_uint32), ("ckpt_bytes", C.c_uint64),
        ("z_bytes", C.c_uint64), ("safe_rerun", C.c_uint32), ("graph", C.c_uint32),
    ]


class ShardC(C.Structure):
    _fields_ = [
        ("chunk_paths", C.c_uint64), ("n_chunks", C.c_uint64),
        ("chunk_begin", C.c_uint64), ("chunk_end", C.c_uint64),
        ("path_begin", C.c_uint64), ("path_end", C.c_uint64),
    ]


def dbl_array(vals: Sequence[float]):
    arr = (C.c_double * max(1, len(vals)))(*[float(v) for v in vals])
    return arr


def u32_array(vals: Sequence[int]):
    return (C.c_uint32 * max(1, len(vals)))(*[int(v) for v in vals])


def i32_array(vals: Sequence[int]):
    return (C.c_int32 * max(1, len(vals)))(*[int(v) for v in vals])


class MarshalledModel:
    """Owns the C arrays a model struct points into."""

    def __init__(self, spec):
        self.keep: List[object] = []
        if isinstance(spec, ModelSpec):
            self.kind = 0
            h, g = spec.heston, spec.grid
            tn, sn, lv = dbl_array(g.t_nodes), dbl_array(g.s_nodes), dbl_array(g.values)
            kinds = i32_array([i.kind for i in spec.instruments])
            strikes = dbl_array([i.strike for i in spec.instruments])
            mats = u32_array([i.maturity_step for i in spec.instruments])
            self.keep += [tn, sn, lv, kinds, strikes, mats]
            self.struct = HestonModelC(
                h.mu, h.s0, h.kappa, h.theta, h.xi, h.rho, h.v0,
                tn, len(g.t_nodes), sn, len(g.s_nodes), lv,
                kinds, strikes, mats, len(spec.instruments),
                spec.mc.steps, spec.mc.dt)
        elif isinstance(spec, BasketSpec):
            self.kind = 1
            s0, chol, sig = dbl_array(spec.s0), dbl_array(spec.chol), dbl_array(spec.sigma)
            assets = u32_array(spec.inst_asset)
            kinds = i32_array([i.kind for i in spec.instruments])
            strikes = dbl_array([i.strike for i in spec.instruments])
            mats = u32_array([i.maturity_step for i in spec.instruments])
            self.keep += [s0, chol, sig, assets, kinds, strikes, mats]
            self.struct = BasketModelC(
                spec.n_assets, s0, spec.r, chol, sig, assets, kinds, strikes, mats,
                len(spec.instruments), spec.steps, spec.dt)
        else:
            raise TypeError("expected ModelSpec or BasketSpec")

    @property
    def ptr(self):
        return C.byref(self.struct)


def num_params(spec) -> int:
    if isinstance(spec, ModelSpec):
        return 5 + len(spec.grid.values)
    return spec.n_assets


def num_outputs(spec) -> int:
    return len(spec.instruments)


def num_randoms(spec) -> int:
    if isinstance(spec, ModelSpec):
        return 2 * spec.mc.steps
    return spec.steps * spec.n_assets
