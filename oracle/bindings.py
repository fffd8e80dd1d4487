"""oracle/bindings.py — TEST INFRASTRUCTURE, NOT PRODUCT CODE.

ctypes bindings of the two CPU checkers:
  * ``Lto``  — oracle/_build/liblto.so, the plain-C restatement (lt_oracle.c);
  * ``Ref``  — oracle/_ref/libltref.so, the unmodified reference library
               compiled in place (ref_driver.cpp).
Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline / reference
arm import this module.
"""
from __future__ import annotations

import ctypes as C
import os
from typing import Optional, Sequence

import numpy as np

from paper_1901_04200_b200.cabi import MarshalledModel, num_outputs, num_params, num_randoms
from paper_1901_04200_b200.model import BasketSpec, ModelSpec

HERE = os.path.dirname(os.path.abspath(__file__))
LTO_PATH = os.path.join(HERE, "_build", "liblto.so")
REF_PATH = os.path.join(HERE, "_ref", "libltref.so")

_dp = C.POINTER(C.c_double)
_u32p = C.POINTER(C.c_uint32)


def _ptr(a: Optional[np.ndarray]):
    if a is None:
        return None
    return a.ctypes.data_as(_dp)


def _arr(x: Sequence[float]) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(x, dtype=np.float64))


class OracleError(RuntimeError):
    def __init__(self, code: int, msg: str = ""):
        super().__init__(f"oracle error {code}: {msg}")
        self.code = code


def build(ref: bool = True) -> None:
    import subprocess
    targets = ["lto"] + (["ref"] if ref and os.path.isdir("/root/reference/proj/include") else [])
    subprocess.check_call(["make", "-s", "-C", HERE] + targets)


class Lto:
    """Plain-C restatement."""

    def __init__(self, path: str = LTO_PATH):
        if not os.path.exists(path):
            build(ref=False)
        self.lib = L = C.CDLL(path)
        L.lto_philox_block.argtypes = [_u32p, _u32p, _u32p]
        L.lto_uniform.argtypes = [C.c_uint32, C.c_uint32]
        L.lto_uniform.restype = C.c_double
        L.lto_inverse_normal_cdf.argtypes = [C.c_double, _dp]
        L.lto_fill_normals.argtypes = [C.c_uint64, C.c_size_t, C.c_int, C.c_uint64, _dp]
        L.lto_heston_path.argtypes = [C.c_void_p, _dp, _dp, _dp, _dp, _dp]
        L.lto_basket_path.argtypes = [C.c_void_p, _dp, _dp, _dp, _dp, _dp]
        L.lto_pass_sums.argtypes = [C.c_int, C.c_void_p, _dp, C.c_uint64, C.c_int, C.c_int,
                                    C.c_uint64, C.c_uint64, _dp, _dp, _dp, _dp]
        L.lto_gradient_of_G.argtypes = [C.c_int, C.c_void_p, _dp, _dp, C.c_uint64, C.c_uint64,
                                        C.c_int, C.c_int, C.c_int, _dp, _dp, _dp, _dp, _dp]

    def philox_block(self, ctr, key):
        c = (C.c_uint32 * 4)(*ctr)
        k = (C.c_uint32 * 2)(*key)
        o = (C.c_uint32 * 4)()
        self.lib.lto_philox_block(c, k, o)
        return list(o)

    def uniform(self, w0, w1):
        return self.lib.lto_uniform(w0, w1)

    def inverse_normal_cdf(self, p):
        out = C.c_double()
        if self.lib.lto_inverse_normal_cdf(p, C.byref(out)):
            raise ValueError("inverse_normal_cdf: p outside (0,1)")
        return out.value

    def fill_normals(self, seed, dim, antithetic, path0, npaths):
        out = np.empty((npaths, dim))
        for i in range(npaths):
            self.lib.lto_fill_normals(seed, dim, int(antithetic), path0 + i, _ptr(out[i]))
        return out

    def path(self, spec, x, z, lam=None):
        mm = MarshalledModel(spec)
        y = np.empty(num_outputs(spec))
        adj = np.empty(num_params(spec)) if lam is not None else None
        fn = self.lib.lto_heston_path if mm.kind == 0 else self.lib.lto_basket_path
        rc = fn(C.cast(mm.ptr, C.c_void_p), _ptr(_arr(x)), _ptr(_arr(z)),
                _ptr(_arr(lam)) if lam is not None else None, _ptr(y), _ptr(adj))
        if rc:
            raise OracleError(rc)
        return y, adj

    def pass_sums(self, spec, x, seed, antithetic=False, lane_width=8, path_offset=0, paths=1,
                  lam=None):
        mm = MarshalledModel(spec)
        xs = _arr(x)
        if lam is None:
            s, s2 = np.empty(num_outputs(spec)), np.empty(num_outputs(spec))
            rc = self.lib.lto_pass_sums(mm.kind, C.cast(mm.ptr, C.c_void_p), _ptr(xs), seed,
                                        int(antithetic), lane_width, path_offset, paths, None,
                                        _ptr(s), _ptr(s2), None)
            if rc:
                raise OracleError(rc)
            return s, s2
        a = np.empty(num_params(spec))
        rc = self.lib.lto_pass_sums(mm.kind, C.cast(mm.ptr, C.c_void_p), _ptr(xs), seed,
                                    int(antithetic), lane_width, path_offset, paths,
                                    _ptr(_arr(lam)), None, None, _ptr(a))
        if rc:
            raise OracleError(rc)
        return a

    def gradient_of_G(self, spec, x, targets, paths, seed, antithetic=False, fresh=False,
                      lane_width=8):
        mm = MarshalledModel(spec)
        m, M = num_outputs(spec), num_params(spec)
        G = C.c_double()
        means, lam, se, grad = np.empty(m), np.empty(m), np.empty(m), np.empty(M)
        rc = self.lib.lto_gradient_of_G(mm.kind, C.cast(mm.ptr, C.c_void_p), _ptr(_arr(x)),
                                        _ptr(_arr(targets)), paths, seed, int(antithetic),
                                        int(fresh), lane_width, C.byref(G), _ptr(means),
                                        _ptr(lam), _ptr(grad), _ptr(se))
        if rc:
            raise OracleError(rc)
        return dict(G=G.value, means=means, lambda_=lam, grad=grad, std_errors=se)

    def estimate_means(self, spec, x, paths, seed, antithetic=False, lane_width=8):
        mm = MarshalledModel(spec)
        m, M = num_outputs(spec), num_params(spec)
        G = C.c_double()
        means, lam, se, grad = np.empty(m), np.empty(m), np.empty(m), np.empty(M)
        rc = self.lib.lto_gradient_of_G(mm.kind, C.cast(mm.ptr, C.c_void_p), _ptr(_arr(x)), None,
                                        paths, seed, int(antithetic), 0, lane_width, C.byref(G),
                                        _ptr(means), _ptr(lam), _ptr(grad), _ptr(se))
        if rc:
            raise OracleError(rc)
        return means, se


class RefProgram:
    def __init__(self, ref: "Ref", handle, spec):
        self.ref, self.h, self.spec = ref, handle, spec
        L = ref.lib
        self.M = L.ltref_num_params(handle)
        self.N = L.ltref_num_randoms(handle)
        self.m = L.ltref_num_outputs(handle)
        self.nodes = L.ltref_num_nodes(handle)

    def __del__(self):
        try:
            self.ref.lib.ltref_free(self.h)
        except Exception:
            pass

    def _chk(self, rc):
        if rc:
            raise OracleError(rc, self.ref.lib.ltref_last_error().decode())

    def initial_params(self):
        x = np.empty(self.M)
        self.ref.lib.ltref_initial_params(self.h, _ptr(x))
        return x

    def gradient_of_G(self, x, targets, paths, seed, antithetic=False, lane_width=8, workers=1,
                      memory_mode=0, fresh=False):
        G = C.c_double()
        means, lam, grad = np.empty(self.m), np.empty(self.m), np.empty(self.M)
        self._chk(self.ref.lib.ltref_gradient_of_G(
            self.h, _ptr(_arr(x)), self.M, _ptr(_arr(targets)), self.m, paths, seed,
            int(antithetic), lane_width, workers, memory_mode, int(fresh), C.byref(G),
            _ptr(means), _ptr(lam), _ptr(grad)))
        return dict(G=G.value, means=means, lambda_=lam, grad=grad)

    def gradient_of_G_space(self, x, targets, draws, lane_width=1):
        draws = _arr(draws)
        G = C.c_double()
        means, lam, grad = np.empty(self.m), np.empty(self.m), np.empty(self.M)
        self._chk(self.ref.lib.ltref_gradient_of_G_space(
            self.h, _ptr(_arr(x)), self.M, _ptr(_arr(targets)), self.m, _ptr(draws),
            draws.size // self.N, lane_width, C.byref(G), _ptr(means), _ptr(lam), _ptr(grad)))
        return dict(G=G.value, means=means, lambda_=lam, grad=grad)

    def gradient_of_G_buffer(self, x, targets, draws, paths, fresh=False, memory_mode=0,
                             lane_width=8, workers=1):
        """gradient_of_G(kernel, x, targets, BufferDrawSource(draws), cfg)"""
        draws = _arr(draws)
        G = C.c_double()
        means, lam, grad = np.empty(self.m), np.empty(self.m), np.empty(self.M)
        self._chk(self.ref.lib.ltref_gradient_of_G_buffer(
            self.h, _ptr(_arr(x)), self.M, _ptr(_arr(targets)), self.m, _ptr(draws),
            draws.size // self.N, paths, int(fresh), memory_mode, lane_width, workers,
            C.byref(G), _ptr(means), _ptr(lam), _ptr(grad)))
        return dict(G=G.value, means=means, lambda_=lam, grad=grad)

    def estimate_means_buffer(self, x, draws, paths, lane_width=8, workers=1):
        draws = _arr(draws)
        means, se = np.empty(self.m), np.empty(self.m)
        self._chk(self.ref.lib.ltref_estimate_means_buffer(
            self.h, _ptr(_arr(x)), self.M, _ptr(draws), draws.size // self.N, paths, lane_width,
            workers, _ptr(means), _ptr(se)))
        return means, se

    def estimate_means(self, x, paths, seed, antithetic=False, lane_width=8, workers=1):
        means, se = np.empty(self.m), np.empty(self.m)
        self._chk(self.ref.lib.ltref_estimate_means(self.h, _ptr(_arr(x)), self.M, paths, seed,
                                                    int(antithetic), lane_width, workers,
                                                    _ptr(means), _ptr(se)))
        return means, se

    def forward_sums(self, x, seed, path_offset, paths, antithetic=False, lane_width=8, workers=1):
        s, s2 = np.empty(self.m), np.empty(self.m)
        self._chk(self.ref.lib.ltref_forward_sums(self.h, _ptr(_arr(x)), self.M, seed,
                                                  int(antithetic), lane_width, workers,
                                                  path_offset, paths, _ptr(s), _ptr(s2)))
        return s, s2

    def reverse_sums(self, x, seed, path_offset, paths, lam, antithetic=False, lane_width=8,
                     workers=1):
        t = np.empty(self.M)
        self._chk(self.ref.lib.ltref_reverse_sums(self.h, _ptr(_arr(x)), self.M, seed,
                                                  int(antithetic), lane_width, workers,
                                                  path_offset, paths, _ptr(_arr(lam)), self.m,
                                                  _ptr(t)))
        return t

    def path_adjoint(self, x, z, lam=None):
        y = np.empty(self.m)
        adj = np.empty(self.M) if lam is not None else None
        self._chk(self.ref.lib.ltref_path_adjoint(
            self.h, _ptr(_arr(x)), self.M, _ptr(_arr(z)), self.N,
            _ptr(_arr(lam)) if lam is not None else None, self.m, _ptr(y), _ptr(adj)))
        return y, adj

    def simulate_path(self, x, z):
        y = np.empty(self.m)
        self._chk(self.ref.lib.ltref_simulate_path(self.h, _ptr(_arr(x)), self.M, _ptr(_arr(z)),
                                                   self.N, _ptr(y)))
        return y

    def finite_diff_gradient_of_G(self, x, targets, paths, seed, h, lane_width=8, workers=1):
        g = np.empty(self.M)
        self._chk(self.ref.lib.ltref_finite_diff_gradient_of_G(
            self.h, _ptr(_arr(x)), self.M, _ptr(_arr(targets)), self.m, paths, seed, lane_width,
            workers, h, _ptr(g)))
        return g


class Ref:
    """The reference library compiled in place (oracle/_ref/libltref.so)."""

    def __init__(self, path: str = REF_PATH):
        if not os.path.exists(path):
            build(ref=True)
        self.lib = L = C.CDLL(path)
        L.ltref_last_error.restype = C.c_char_p
        L.ltref_philox_block.argtypes = [_u32p, _u32p, _u32p]
        L.ltref_uniform.argtypes = [C.c_uint32, C.c_uint32]
        L.ltref_uniform.restype = C.c_double
        L.ltref_inverse_normal_cdf.argtypes = [C.c_double, _dp]
        L.ltref_fill_normals.argtypes = [C.c_uint64, C.c_size_t, C.c_int, C.c_uint64, C.c_uint64,
                                         _dp]
        for name in ("ltref_record_heston", "ltref_record_basket"):
            getattr(L, name).argtypes = [C.c_void_p]
            getattr(L, name).restype = C.c_void_p
        L.ltref_record_linear.restype = C.c_void_p
        L.ltref_free.argtypes = [C.c_void_p]
        for name in ("ltref_num_params", "ltref_num_randoms", "ltref_num_outputs",
                     "ltref_num_nodes"):
            getattr(L, name).argtypes = [C.c_void_p]
            getattr(L, name).restype = C.c_size_t
        L.ltref_initial_params.argtypes = [C.c_void_p, _dp]
        sz, u64, i = C.c_size_t, C.c_uint64, C.c_int
        L.ltref_gradient_of_G.argtypes = [C.c_void_p, _dp, sz, _dp, sz, u64, u64, i, i, i, i, i,
                                          _dp, _dp, _dp, _dp]
        L.ltref_gradient_of_G_space.argtypes = [C.c_void_p, _dp, sz, _dp, sz, _dp, sz, i, _dp,
                                                _dp, _dp, _dp]
        L.ltref_estimate_means.argtypes = [C.c_void_p, _dp, sz, u64, u64, i, i, i, _dp, _dp]
        L.ltref_gradient_of_G_buffer.argtypes = [C.c_void_p, _dp, sz, _dp, sz, _dp, sz, u64, i,
                                                 i, i, i, _dp, _dp, _dp, _dp]
        L.ltref_estimate_means_buffer.argtypes = [C.c_void_p, _dp, sz, _dp, sz, u64, i, i, _dp,
                                                  _dp]
        L.ltref_forward_sums.argtypes = [C.c_void_p, _dp, sz, u64, i, i, i, u64, u64, _dp, _dp]
        L.ltref_reverse_sums.argtypes = [C.c_void_p, _dp, sz, u64, i, i, i, u64, u64, _dp, sz,
                                         _dp]
        L.ltref_path_adjoint.argtypes = [C.c_void_p, _dp, sz, _dp, sz, _dp, sz, _dp, _dp]
        L.ltref_simulate_path.argtypes = [C.c_void_p, _dp, sz, _dp, sz, _dp]
        L.ltref_finite_diff_gradient_of_G.argtypes = [C.c_void_p, _dp, sz, _dp, sz, u64, u64, i,
                                                      i, C.c_double, _dp]

    def philox_block(self, ctr, key):
        c = (C.c_uint32 * 4)(*ctr)
        k = (C.c_uint32 * 2)(*key)
        o = (C.c_uint32 * 4)()
        self.lib.ltref_philox_block(c, k, o)
        return list(o)

    def uniform(self, w0, w1):
        return self.lib.ltref_uniform(w0, w1)

    def inverse_normal_cdf(self, p):
        out = C.c_double()
        if self.lib.ltref_inverse_normal_cdf(p, C.byref(out)):
            raise ValueError(self.lib.ltref_last_error().decode())
        return out.value

    def fill_normals(self, seed, dim, antithetic, path0, npaths):
        out = np.empty((npaths, dim))
        rc = self.lib.ltref_fill_normals(seed, dim, int(antithetic), path0, npaths, _ptr(out))
        if rc:
            raise OracleError(rc, self.lib.ltref_last_error().decode())
        return out

    def program(self, spec) -> RefProgram:
        mm = MarshalledModel(spec)
        fn = self.lib.ltref_record_heston if mm.kind == 0 else self.lib.ltref_record_basket
        h = fn(C.cast(mm.ptr, C.c_void_p))
        if not h:
            raise OracleError(1, self.lib.ltref_last_error().decode())
        return RefProgram(self, h, spec)

    def linear_program(self) -> RefProgram:
        return RefProgram(self, self.lib.ltref_record_linear(), None)


def ref_available() -> bool:
    return os.path.exists(REF_PATH) or os.path.isdir("/root/reference/proj/include")
