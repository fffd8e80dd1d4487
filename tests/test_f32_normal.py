"""The fp32 mode's inverse normal (rng.cuh gen_segment<float>, f32_normal.h)
restated in numpy float32 — q from the top 23 bits of the 52-bit uniform,
min(p, 1-p) from the 52-bit integer for tail slots, the fitted rationals —
against the fp64 inverse normal of the same Philox uniforms. The SFU's
approximate log2 / rsqrt / reciprocal are replaced by correctly rounded float
operations here, so the bar (1e-6 relative, 2e-7 absolute near 0) leaves room
for their few ulp."""
import os
import re

import numpy as np
from scipy.special import ndtri

HDR = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                   "paper_1901_04200_b200", "csrc", "f32_normal.h")


def coeffs():
    src = open(HDR).read()
    out = {}
    for name, body in re.findall(r"constexpr float (\w+)\(int k\) \{\s*return (.*?);\s*\}", src,
                                 re.S):
        out[name] = [np.float32(float(v.rstrip("f"))) for v in
                     re.findall(r"(-?\d\.\d+e[+-]\d+f)", body)]
    return out


def horner(c, x):
    acc = np.full_like(x, c[-1])
    for k in range(len(c) - 2, -1, -1):
        acc = (acc * x + c[k]).astype(np.float32)
    return acc


def f32_normals(hi, lo, c):
    """the kernel's float mapping of Philox words (hi, lo) -> z"""
    hi, lo = hi.astype(np.uint64), lo.astype(np.uint64)
    u = (hi >> np.uint64(9)).astype(np.float32)
    q = (u * np.float32(2.0 ** -23) + np.float32(2.0 ** -24 - 0.5)).astype(np.float32)
    tail = np.abs(q) > np.float32(0.425)
    r = (np.float32(0.180625) - q * q).astype(np.float32)
    num = horner(c["central_num"], r)
    den = horner([np.float32(1.0)] + c["central_den"], r)
    z = (q * num / den).astype(np.float32)
    flip = np.where(hi >> np.uint64(31), np.uint64(0x3FFFFFF), np.uint64(0))
    ka = (hi >> np.uint64(6)) ^ flip
    kb = (lo >> np.uint64(6)) ^ flip
    rr = (ka.astype(np.float32) * np.float32(2.0 ** -26) +
          (2 * kb + 1).astype(np.float32) * np.float32(2.0 ** -53)).astype(np.float32)
    sq = np.sqrt(-np.log(rr.astype(np.float64))).astype(np.float32)
    t1 = (sq - np.float32(1.6)).astype(np.float32)
    t2 = (sq - np.float32(5.0)).astype(np.float32)
    zt = np.where(sq <= 5.0,
                  horner(c["tail1_num"], t1) / horner([np.float32(1.0)] + c["tail1_den"], t1),
                  horner(c["tail2_num"], t2) / horner([np.float32(1.0)] + c["tail2_den"], t2))
    zt = np.where(hi >> np.uint64(31), zt, -zt)
    return np.where(tail, zt, z).astype(np.float32)


def test_fp32_inverse_normal_against_fp64():
    c = coeffs()
    assert sorted(c) == sorted(["central_num", "central_den", "tail1_num", "tail1_den",
                                "tail2_num", "tail2_den"])
    g = np.random.default_rng(7)
    hi = g.integers(0, 2 ** 32, 2_000_000, dtype=np.uint64)
    lo = g.integers(0, 2 ** 32, 2_000_000, dtype=np.uint64)
    # the generator's extremes and the deep tails (r > 5 row: a = hi >> 6 tiny)
    hi[:6] = [0, 63, 2 ** 32 - 1, 2 ** 32 - 64, 1 << 31, (1 << 31) - 1]
    lo[:6] = [0, 2 ** 32 - 1, 2 ** 32 - 1, 0, 0, 2 ** 32 - 1]
    hi[6:20000] = g.integers(0, 64 << 6, 19994)
    n = ((hi >> np.uint64(6)) << np.uint64(26)) | (lo >> np.uint64(6))
    p = (2.0 * n.astype(np.float64) + 1.0) * 2.0 ** -53  # uniform_from_bits
    want = ndtri(p)
    got = f32_normals(hi, lo, c).astype(np.float64)
    err = np.abs(got - want) / np.maximum(np.abs(want), 0.2)
    assert np.max(err) <= 1e-6, (np.max(err), p[np.argmax(err)])
    assert np.all(np.sign(got) == np.sign(want))
