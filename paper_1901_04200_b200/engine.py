"""Python binding of the CUDA engine's C ABI (include/lanetape_b200.h).

Mirrors the reference's calling surface (expectation.hpp): ``gradient_of_G``,
``estimate_means``, ``finite_diff_gradient_of_G`` returning ``GradientReport`` /
``MeansResult``; ``Objective`` factories for the reference's calibrator
(calibrate.hpp:117-120). There is no CPU fallback: if the built library
(``_lib/liblanetape_b200.so``) is missing or no sm_100 GPU is usable, every
call raises.
"""
from __future__ import annotations

import ctypes as C
import os
from typing import Optional, Sequence

import numpy as np

from . import cabi
from .cabi import (LTG_ECUDA, LTG_EINVAL, LTG_ENUMERIC, DrawsC, MarshalledModel, MCConfigC,
                   ReportC, ShardC, TimingC)
from .model import (BufferDrawSource, GradientReport, MCConfig, MeansResult, SampleSpace,
                    memory_mode_name)

LIB_PATH = os.environ.get("LTG_LIB") or os.path.join(
    os.path.dirname(os.path.abspath(__file__)), "_lib", "liblanetape_b200.so")

_dp = C.POINTER(C.c_double)


class EvalError(RuntimeError):
    """Numerical failure (the reference's lanetape::EvalError)."""


class EngineError(RuntimeError):
    """CUDA / NCCL failure."""


_lib = None


def load_library(path: str = LIB_PATH):
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise EngineError(f"CUDA engine library not built: {path} (run __graft_entry__.build())")
    L = C.CDLL(path)
    L.ltg_abi_version.restype = C.c_int
    L.ltg_create_heston.argtypes = [C.c_void_p, C.c_int, C.POINTER(C.c_void_p)]
    L.ltg_create_basket.argtypes = [C.c_void_p, C.c_int, C.POINTER(C.c_void_p)]
    L.ltg_create_heston_devices.argtypes = [C.c_void_p, C.POINTER(C.c_int), C.c_int,
                                            C.POINTER(C.c_void_p)]
    L.ltg_create_basket_devices.argtypes = L.ltg_create_heston_devices.argtypes
    L.ltg_destroy.argtypes = [C.c_void_p]
    L.ltg_last_error.argtypes = [C.c_void_p]
    L.ltg_last_error.restype = C.c_char_p
    for f in ("ltg_num_params", "ltg_num_outputs", "ltg_num_randoms"):
        getattr(L, f).argtypes = [C.c_void_p]
        getattr(L, f).restype = C.c_size_t
    L.ltg_pack_params.argtypes = [C.c_void_p, _dp, C.c_size_t]
    L.ltg_gradient_of_G.argtypes = [C.c_void_p, _dp, C.c_size_t, _dp, C.c_size_t,
                                    C.POINTER(MCConfigC), C.POINTER(ReportC)]
    L.ltg_gradient_of_G_tangent.argtypes = L.ltg_gradient_of_G.argtypes
    L.ltg_estimate_means.argtypes = [C.c_void_p, _dp, C.c_size_t, C.POINTER(MCConfigC), _dp, _dp]
    L.ltg_gradient_of_G_draws.argtypes = [C.c_void_p, _dp, C.c_size_t, _dp, C.c_size_t,
                                          C.POINTER(DrawsC), C.POINTER(MCConfigC),
                                          C.POINTER(ReportC)]
    L.ltg_estimate_means_draws.argtypes = [C.c_void_p, _dp, C.c_size_t, C.POINTER(DrawsC),
                                           C.c_uint64, _dp, _dp]
    L.ltg_finite_diff_gradient_of_G.argtypes = [C.c_void_p, _dp, C.c_size_t, _dp, C.c_size_t,
                                                C.POINTER(MCConfigC), C.c_double, _dp]
    L.ltg_fill_normals.argtypes = [C.c_void_p, C.c_uint64, C.c_size_t, C.c_int, C.c_uint64,
                                   C.c_uint64, _dp]
    L.ltg_inverse_normal.argtypes = [C.c_void_p, _dp, C.c_size_t, _dp]
    L.ltg_chunk_sums.argtypes = [C.c_void_p, _dp, C.c_size_t, _dp, C.c_size_t, C.c_uint64,
                                 C.c_int, C.c_uint64, C.c_uint64, _dp, _dp, _dp]
    L.ltg_last_timing.argtypes = [C.c_void_p, C.POINTER(TimingC)]
    L.ltg_set_hbm_budget.argtypes = [C.c_void_p, C.c_uint64]
    L.ltg_set_timing.argtypes = [C.c_void_p, C.c_int]
    L.ltg_path_payoffs.argtypes = [C.c_void_p, _dp, C.c_size_t, C.c_uint64, C.c_int, C.c_uint64,
                                   C.c_uint64, _dp]
    L.ltg_rng_exact.argtypes = [C.c_void_p]
    L.ltg_shard_plan.argtypes = [C.c_uint64, C.c_int, C.c_int, C.POINTER(ShardC)]
    L.ltg_nccl_unique_id.argtypes = [C.c_char_p]
    L.ltg_attach_nccl.argtypes = [C.c_void_p, C.c_char_p, C.c_int, C.c_int]
    L.ltg_probe_fp64_rate.argtypes = [C.c_int, _dp, _dp]
    L.ltg_probe_fp32_rate.argtypes = [C.c_int, _dp]
    L.ltg_rng_selftest.argtypes = [C.c_uint64, C.POINTER(C.c_uint64), C.POINTER(C.c_int)]
    _lib = L
    return L


def probe_fp64_rate(device: int = 0) -> float:
    """Measured FP64 issue rate (thread FP64 instructions/s) of the GPU."""
    L = load_library()
    r, clk = C.c_double(), C.c_double()
    if L.ltg_probe_fp64_rate(device, C.byref(r), C.byref(clk)):
        raise EngineError("fp64 probe failed")
    return r.value


def probe_fp32_rate(device: int = 0) -> float:
    """Measured FP32 FFMA issue rate (thread instructions/s) of the GPU."""
    L = load_library()
    r = C.c_double()
    if L.ltg_probe_fp32_rate(device, C.byref(r)):
        raise EngineError("fp32 probe failed")
    return r.value


def rng_selftest(n: int = 1 << 20):
    """Host-only check of the GPU log restatement against this host's libm."""
    L = load_library()
    bad, exact = C.c_uint64(), C.c_int()
    rc = L.ltg_rng_selftest(n, C.byref(bad), C.byref(exact))
    return {"found": rc == 0, "mismatches": bad.value, "exact": bool(exact.value)}


def _arr(x: Sequence[float]) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(x, dtype=np.float64))


def _p(a: Optional[np.ndarray]):
    return None if a is None else a.ctypes.data_as(_dp)


def _cfg(cfg: MCConfig) -> MCConfigC:
    return MCConfigC(int(cfg.paths), int(cfg.seed) & 0xFFFFFFFFFFFFFFFF, int(bool(cfg.antithetic)),
                     int(bool(cfg.fresh_step2_paths)), int(cfg.memory_mode), int(cfg.precision))


def shard_plan(paths: int, rank: int, world: int) -> dict:
    L = load_library()
    s = ShardC()
    rc = L.ltg_shard_plan(paths, rank, world, C.byref(s))
    if rc:
        raise ValueError("shard_plan: bad arguments")
    return {k: getattr(s, k) for k, _ in ShardC._fields_}


def nccl_unique_id() -> bytes:
    L = load_library()
    buf = C.create_string_buffer(128)
    if L.ltg_nccl_unique_id(buf):
        raise EngineError(L.ltg_last_error(None).decode())
    return buf.raw


class Engine:
    """A model bound to one GPU: the GPU counterpart of a recorded program
    (record_heston_program(ModelSpec) for Heston-SLV; the config-4 basket)."""

    def __init__(self, spec, device: int = 0, devices: Optional[Sequence[int]] = None):
        """devices: a single-process multi-GPU context over these devices
        (ltg_create_*_devices); otherwise one context on `device`."""
        self.lib = load_library()
        self.spec = spec
        self._mm = MarshalledModel(spec)
        h = C.c_void_p()
        model = C.cast(self._mm.ptr, C.c_void_p)
        if devices is not None:
            devs = (C.c_int * len(devices))(*devices)
            fn = (self.lib.ltg_create_heston_devices if self._mm.kind == 0
                  else self.lib.ltg_create_basket_devices)
            rc = fn(model, devs, len(devices), C.byref(h))
        else:
            fn = self.lib.ltg_create_heston if self._mm.kind == 0 else self.lib.ltg_create_basket
            rc = fn(model, device, C.byref(h))
        if rc:
            msg = self.lib.ltg_last_error(None).decode()
            raise (ValueError if rc == LTG_EINVAL else EngineError)(msg)
        self.h = h
        self.M = self.lib.ltg_num_params(h)
        self.m = self.lib.ltg_num_outputs(h)
        self.N = self.lib.ltg_num_randoms(h)

    def close(self):
        if getattr(self, "h", None):
            self.lib.ltg_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _raise(self, rc: int):
        msg = self.lib.ltg_last_error(self.h).decode()
        if rc == LTG_EINVAL:
            raise ValueError(msg)
        if rc == LTG_ENUMERIC:
            raise EvalError(msg)
        raise EngineError(msg)

    @property
    def rng_exact(self) -> bool:
        return bool(self.lib.ltg_rng_exact(self.h))

    def pack_params(self) -> np.ndarray:
        x = np.empty(self.M)
        self.lib.ltg_pack_params(self.h, _p(x), self.M)
        return x

    @staticmethod
    def _draws(source):
        """(ltg_draws, keep-alive array) of a BufferDrawSource / SampleSpace"""
        if isinstance(source, SampleSpace):
            buf = np.ascontiguousarray(source.draws, dtype=np.float64).ravel()
            if buf.size != source.scenarios * source.num_randoms:
                raise ValueError("SampleSpace: draws size does not match dimensions")
            return DrawsC(_p(buf), source.scenarios, source.num_randoms), buf
        if isinstance(source, BufferDrawSource):
            return DrawsC(_p(source.draws), source.paths(), source.dimension()), source.draws
        raise TypeError("source must be a BufferDrawSource or a SampleSpace")

    def gradient_of_G(self, x, targets, cfg, std_errors: bool = False,
                      method: str = "adjoint", source=None) -> GradientReport:
        """expectation.hpp:346-351 (Philox draws from cfg.seed). method="adjoint"
        is the reference's two-pass scheme; "tangent" replaces pass 2 by
        pathwise forward tangents (ltg_gradient_of_G_tangent: small-M Heston
        models only).

        The reference's other overloads (ltg_gradient_of_G_draws):
        ``source=BufferDrawSource`` is gradient_of_G(kernel, params, targets,
        src, cfg) (:300-344); ``cfg=SampleSpace`` is the scenario-set overload
        (:354-367: paths = scenarios, seed 0, recompute)."""
        xa, ta = _arr(x), _arr(targets)
        means, lam, grad = np.empty(self.m), np.empty(self.m), np.empty(self.M)
        se = np.empty(self.m) if std_errors else None
        rep = ReportC(0.0, _p(means), _p(lam), _p(grad), _p(se), 0, 0, 0)
        if method not in ("adjoint", "tangent"):
            raise ValueError(f"unknown method {method!r}")
        if isinstance(cfg, SampleSpace):
            source, cfg = cfg, MCConfig(paths=cfg.scenarios, seed=0)
        c = _cfg(cfg)
        if source is not None:
            if method != "adjoint":
                raise ValueError("caller draws: method='adjoint' only")
            d, keep = self._draws(source)
            rc = self.lib.ltg_gradient_of_G_draws(self.h, _p(xa), xa.size, _p(ta), ta.size,
                                                  C.byref(d), C.byref(c), C.byref(rep))
            del keep
        else:
            fn = (self.lib.ltg_gradient_of_G if method == "adjoint"
                  else self.lib.ltg_gradient_of_G_tangent)
            rc = fn(self.h, _p(xa), xa.size, _p(ta), ta.size, C.byref(c), C.byref(rep))
        if rc:
            self._raise(rc)
        out = GradientReport(rep.G, means.tolist(), lam.tolist(), grad.tolist(), int(rep.paths),
                             memory_mode_name(rep.mode), int(rep.seed))
        if std_errors:
            out.std_errors = se.tolist()
        return out

    def prepared_gradient(self, x, targets, cfg: MCConfig):
        """A bound ltg_gradient_of_G call on fixed host buffers (what a C / C++
        caller of the ABI holds): returns (call, xbuf, tbuf, out) where call()
        runs the two-pass gradient on the current contents of the host
        arrays xbuf / tbuf and leaves G, means, lambda and grad in `out`
        (bench.py's end-to-end timing: no per-call Python marshalling)."""
        xb, tb = _arr(x).copy(), _arr(targets).copy()
        out = {"means": np.empty(self.m), "lambda": np.empty(self.m), "grad": np.empty(self.M)}
        rep = ReportC(0.0, _p(out["means"]), _p(out["lambda"]), _p(out["grad"]), None, 0, 0, 0)
        c = _cfg(cfg)
        fn, h, lib = self.lib.ltg_gradient_of_G, self.h, self
        args = (h, _p(xb), xb.size, _p(tb), tb.size, C.byref(c), C.byref(rep))

        def call():
            rc = fn(*args)
            if rc:
                lib._raise(rc)
            return rep.G

        out["report"] = rep
        return call, xb, tb, out

    def estimate_means(self, x, cfg, source=None, paths: Optional[int] = None) -> MeansResult:
        """expectation.hpp:281-286 (Philox draws from cfg.seed); with
        ``source=BufferDrawSource`` and ``paths`` the PathDrawSource overload
        (:274-279), with ``cfg=SampleSpace`` the scenario-set overload
        (:287-294) — both through ltg_estimate_means_draws."""
        xa = _arr(x)
        means, se = np.empty(self.m), np.empty(self.m)
        if isinstance(cfg, SampleSpace):
            source, paths = cfg, cfg.scenarios
        if source is not None:
            if paths is None:
                raise ValueError("estimate_means with a draw source needs paths")
            d, keep = self._draws(source)
            rc = self.lib.ltg_estimate_means_draws(self.h, _p(xa), xa.size, C.byref(d), paths,
                                                   _p(means), _p(se))
            del keep
        else:
            paths = cfg.paths
            c = _cfg(cfg)
            rc = self.lib.ltg_estimate_means(self.h, _p(xa), xa.size, C.byref(c), _p(means),
                                             _p(se))
        if rc:
            self._raise(rc)
        return MeansResult(means.tolist(), se.tolist(), int(paths))

    def finite_diff_gradient_of_G(self, x, targets, cfg: MCConfig, h: float) -> np.ndarray:
        """expectation.hpp:372-400"""
        xa, ta = _arr(x), _arr(targets)
        g = np.empty(self.M)
        c = _cfg(cfg)
        rc = self.lib.ltg_finite_diff_gradient_of_G(self.h, _p(xa), xa.size, _p(ta), ta.size,
                                                    C.byref(c), h, _p(g))
        if rc:
            self._raise(rc)
        return g

    def fill_normals(self, seed: int, dim: int, antithetic: bool, path0: int,
                     npaths: int) -> np.ndarray:
        """PhiloxNormalSource(seed, dim, antithetic).fill(p) for p in [path0, path0+npaths)."""
        out = np.empty((npaths, dim))
        rc = self.lib.ltg_fill_normals(self.h, seed, dim, int(antithetic), path0, npaths, _p(out))
        if rc:
            self._raise(rc)
        return out

    def chunk_sums(self, x, lam, seed: int, antithetic: bool, path0: int, npaths: int):
        """(Σy, Σy², adjoint total) over global paths [path0, path0+npaths): one
        chunk of forward_pass / reverse_pass (expectation.hpp:152-249) seeded
        with the given lambda."""
        xa, la = _arr(x), _arr(lam)
        s1, s2, adj = np.empty(self.m), np.empty(self.m), np.empty(self.M)
        rc = self.lib.ltg_chunk_sums(self.h, _p(xa), xa.size, _p(la), la.size, seed,
                                     int(antithetic), path0, npaths, _p(s1), _p(s2), _p(adj))
        if rc:
            self._raise(rc)
        return s1, s2, adj

    def inverse_normal(self, p) -> np.ndarray:
        """inverse_normal_cdf(p) elementwise on the GPU (rng.hpp:45-85); p of the
        generator's form (2k+1)*2^-53 in (0, 1)."""
        pa = _arr(p)
        z = np.empty(pa.size)
        rc = self.lib.ltg_inverse_normal(self.h, _p(pa), pa.size, _p(z))
        if rc:
            self._raise(rc)
        return z

    def path_payoffs(self, x, seed: int, antithetic: bool, path0: int, npaths: int) -> np.ndarray:
        """Per-path program outputs for the draws of paths [path0, path0+npaths)."""
        xa = _arr(x)
        y = np.empty((npaths, self.m))
        rc = self.lib.ltg_path_payoffs(self.h, _p(xa), xa.size, seed, int(antithetic), path0,
                                       npaths, _p(y))
        if rc:
            self._raise(rc)
        return y

    def set_hbm_budget(self, nbytes: int) -> None:
        """Cap the HBM held for checkpoints + draw store (0: free memory)."""
        rc = self.lib.ltg_set_hbm_budget(self.h, int(nbytes))
        if rc:
            self._raise(rc)

    def set_timing(self, on: bool) -> None:
        """Device timing events of the calls (ltg_set_timing; on by default):
        off takes the events out of a small call's critical path, and
        timing() then reports zero device times."""
        rc = self.lib.ltg_set_timing(self.h, 1 if on else 0)
        if rc:
            self._raise(rc)

    def timing(self) -> dict:
        t = TimingC()
        self.lib.ltg_last_timing(self.h, C.byref(t))
        return {k: getattr(t, k) for k, _ in TimingC._fields_}

    def attach_nccl(self, uid: bytes, rank: int, world: int) -> None:
        rc = self.lib.ltg_attach_nccl(self.h, uid, rank, world)
        if rc:
            self._raise(rc)

    # ---- calibrate.hpp:117-120 plug point ----
    def objective(self, targets, cfg: MCConfig):
        """(value_and_grad, value) callbacks for the reference's gradient_descent
        under common random numbers (every call replays cfg.seed)."""
        ta = list(targets)

        def value_and_grad(x):
            return self.gradient_of_G(x, ta, cfg)

        def value(x):
            means = self.estimate_means(x, cfg).means
            g = 0.0
            for mv, t in zip(means, ta):
                l = mv - t
                g += 0.5 * l * l
            return g

        return value_and_grad, value
