"""The five BASELINE.json configurations expressed through the reference API.

Configs 1-3 and 5 are instances of the reference's own Heston-SLV program
(record_heston_program, heston.hpp:245-325) via the embedding of SURVEY.md
§8(d): a GBM / local-vol model is Heston with kappa = xi = rho = 0,
theta = v0 = 1 (so V == 1 exactly and sqrt(V) == 1) and the volatility carried
by the leverage grid. Config 4 (16-asset correlated GBM) has no model in the
reference layer; it is the basket program of oracle/ref_driver.cpp.

Everything BASELINE.json leaves open is fixed here, seeded and documented
(DESIGN.md §3): seeds, cfg2 r and s0, cfg3 strike spacing, cfg4 S0/r/eval
point/correlation, and the generator for "true values drawn from the seed"
(Philox4x32-10 counter (i, 0, 0, 'conf') under the config seed, mapped with
the reference's uniform_from_bits).
"""
from __future__ import annotations

import json
import math
import os
from dataclasses import dataclass, field
from typing import List, Optional

from .model import (CALL, BasketSpec, HestonParams, Instrument, LeverageGrid, McSettings,
                    ModelSpec)

HERE = os.path.dirname(os.path.abspath(__file__))
TARGETS_DIR = os.path.join(HERE, "configs")

GRAD_SEED = 42          # seed of the paths the gradient is evaluated on
TARGET_SEED = 4242      # separate seed of the target-generating forward runs
TARGET_PATHS = 1 << 22


def _philox4x32(ctr, key):
    """Philox4x32-10 (rng.hpp:19-31), for seeded config values only."""
    c = list(ctr)
    k0, k1 = key
    for _ in range(10):
        p0 = 0xD2511F53 * c[0]
        p1 = 0xCD9E8D57 * c[2]
        c = [((p1 >> 32) ^ c[1] ^ k0) & 0xFFFFFFFF, p1 & 0xFFFFFFFF,
             ((p0 >> 32) ^ c[3] ^ k1) & 0xFFFFFFFF, p0 & 0xFFFFFFFF]
        k0 = (k0 + 0x9E3779B9) & 0xFFFFFFFF
        k1 = (k1 + 0xBB67AE85) & 0xFFFFFFFF
    return c


def seeded_uniform(seed: int, i: int) -> float:
    w = _philox4x32([i & 0xFFFFFFFF, i >> 32, 0, 0x636F6E66], [seed & 0xFFFFFFFF, seed >> 32])
    return ((w[0] >> 6) * 67108864.0 + (w[1] >> 6) + 0.5) * (1.0 / 4503599627370496.0)


def normal_cdf(x: float) -> float:
    return 0.5 * math.erfc(-x / math.sqrt(2.0))


def bs_call_undiscounted(s0, strike, sigma, T, mu):
    """tests/support/oracles.hpp:28-34 (undiscounted, like the reference payoffs)."""
    F = s0 * math.exp(mu * T)
    sd = sigma * math.sqrt(T)
    d1 = (math.log(F / strike) + 0.5 * sd * sd) / sd
    return F * normal_cdf(d1) - strike * normal_cdf(d1 - sd)


@dataclass
class BenchConfig:
    name: str
    spec: object                 # ModelSpec or BasketSpec
    x: List[float]               # evaluation point (packed)
    truth: List[float]           # truth the targets come from (packed)
    paths: int
    seed: int = GRAD_SEED
    targets: Optional[List[float]] = None
    target_kind: str = "mc"      # "mc" (separate-seed forward run) or "bs" (closed form)
    description: str = ""
    grad_index: List[int] = field(default_factory=list)  # BASELINE's M params inside grad

    @property
    def M(self):
        return len(self.x)

    @property
    def m(self):
        return len(self.spec.instruments)


def _lv_params(mu: float, s0: float) -> HestonParams:
    # GBM / local vol embedding: V == 1, sqrt(V) == 1, vol lives in the grid
    return HestonParams(mu=mu, kappa=0.0, theta=1.0, xi=0.0, rho=0.0, v0=1.0, s0=s0)


def cfg1() -> BenchConfig:
    steps, dt = 16, 1.0 / 16
    strikes = [80, 90, 100, 110, 120, 85, 100, 115]
    mats = [4, 4, 4, 8, 8, 16, 16, 16]
    grid = LeverageGrid([0.0, 0.25, 0.5, 0.75], [0.0], [0.25] * 4)
    spec = ModelSpec(_lv_params(0.02, 100.0), grid,
                     [Instrument(CALL, float(k), m) for k, m in zip(strikes, mats)],
                     McSettings(1 << 16, steps, dt, GRAD_SEED))
    true_sig = [0.20, 0.22, 0.25, 0.23]
    x = [0.0, 1.0, 0.0, 0.0, 1.0] + [0.25] * 4
    truth = [0.0, 1.0, 0.0, 0.0, 1.0] + true_sig
    targets = []
    for k, ms in zip(strikes, mats):
        T = ms * dt
        nb = int(round(T / 0.25))
        var = sum(s * s for s in true_sig[:nb]) / nb
        targets.append(bs_call_undiscounted(100.0, float(k), math.sqrt(var), T, 0.02))
    return BenchConfig("cfg1_gbm", spec, x, truth, 1 << 16, targets=targets, target_kind="bs",
                       description="GBM, piecewise-constant vol (4), 8 calls, 16 steps, 2^16 paths",
                       grad_index=list(range(5, 9)))


def cfg2() -> BenchConfig:
    steps, dt = 64, 1.0 / 64
    t_nodes = [0.125 * i for i in range(8)]
    s_nodes = [0.0, 70.0, 90.0, 110.0, 130.0]
    true_vols = [0.15 + 0.2 * seeded_uniform(2002, i) for i in range(40)]
    ins = [Instrument(CALL, float(k), 8 * (j + 1)) for j in range(8)
           for k in (80, 90, 100, 110, 120)]
    spec = ModelSpec(_lv_params(0.02, 100.0), LeverageGrid(t_nodes, s_nodes, [0.25] * 40), ins,
                     McSettings(1 << 20, steps, dt, GRAD_SEED))
    base = [0.0, 1.0, 0.0, 0.0, 1.0]
    return BenchConfig("cfg2_localvol", spec, base + [0.25] * 40, base + true_vols, 1 << 20,
                       description="local-vol 8x5 grid (40), 40 calls, 64 steps, 2^20 paths",
                       grad_index=list(range(5, 45)))


def _heston_spec(paths: int) -> ModelSpec:
    steps, dt = 756, 1.0 / 252
    mats = [63, 126, 252, 378, 504, 756]
    strikes = [70.0 + 60.0 * j / 9.0 for j in range(10)]
    ins = [Instrument(CALL, k, ms) for ms in mats for k in strikes]
    hp = HestonParams(mu=0.01, kappa=2.0, theta=0.05, xi=0.4, rho=-0.5, v0=0.05, s0=100.0)
    return ModelSpec(hp, LeverageGrid([0.0], [0.0], [1.0]), ins, McSettings(paths, steps, dt,
                                                                             GRAD_SEED))


def cfg3() -> BenchConfig:
    return BenchConfig("cfg3_heston", _heston_spec(1 << 20), [2.0, 0.05, 0.4, -0.5, 0.05, 1.0],
                       [1.5, 0.04, 0.5, -0.7, 0.04, 1.0], 1 << 20,
                       description="Heston full-truncation Euler, 756 steps, 60 calls, 2^20 paths",
                       grad_index=list(range(5)))


def cfg5(paths: int = 1 << 26) -> BenchConfig:
    c = cfg3()
    c.name = "cfg5_heston_scaling"
    c.spec = _heston_spec(paths)
    c.paths = paths
    c.description = f"config 3 at {paths} paths"
    c.targets = None
    return c


def cholesky(a: List[List[float]]) -> List[List[float]]:
    """Plain Cholesky in a fixed loop order (bitwise reproducible)."""
    n = len(a)
    L = [[0.0] * n for _ in range(n)]
    for i in range(n):
        for j in range(i + 1):
            s = a[i][j]
            for k in range(j):
                s -= L[i][k] * L[j][k]
            L[i][j] = math.sqrt(s) if i == j else s / L[j][j]
    return L


def basket_correlation(n: int = 16, seed: int = 4005) -> List[List[float]]:
    """A = B B^T + n I with B_ij ~ U(-1, 1) from the seed, scaled to unit diagonal."""
    B = [[2.0 * seeded_uniform(seed, i * n + j) - 1.0 for j in range(n)] for i in range(n)]
    A = [[sum(B[i][k] * B[j][k] for k in range(n)) + (n if i == j else 0.0) for j in range(n)]
         for i in range(n)]
    return [[A[i][j] / math.sqrt(A[i][i] * A[j][j]) for j in range(n)] for i in range(n)]


def cfg4(paths: int = 1 << 22) -> BenchConfig:
    n, steps, dt, r = 16, 50, 1.0 / 50, 0.02
    corr = basket_correlation(n)
    L = cholesky(corr)
    chol = [L[i][j] for i in range(n) for j in range(n)]
    true_sig = [0.15 + 0.25 * seeded_uniform(4004, a) for a in range(n)]
    ins, assets = [], []
    for a in range(n):
        for k in (90.0, 100.0, 110.0):
            ins.append(Instrument(CALL, k, steps))
            assets.append(a)
    spec = BasketSpec([100.0] * n, r, chol, [0.25] * n, ins, assets, steps, dt)
    targets = [bs_call_undiscounted(100.0, i.strike, true_sig[a], 1.0, r)
               for i, a in zip(ins, assets)]
    return BenchConfig("cfg4_basket16", spec, [0.25] * n, true_sig, paths, targets=targets,
                       target_kind="bs",
                       description="16-asset correlated GBM, 48 calls, 50 steps, 2^22 paths",
                       grad_index=list(range(n)))


ALL = {"cfg1": cfg1, "cfg2": cfg2, "cfg3": cfg3, "cfg4": cfg4, "cfg5": cfg5}


def targets_path(name: str) -> str:
    return os.path.join(TARGETS_DIR, f"{name}_targets.json")


def load_targets(cfg: BenchConfig) -> Optional[List[float]]:
    """Committed targets of the separate-seed forward runs (tools/make_targets.py,
    computed with the reference library itself)."""
    if cfg.targets is not None:
        return cfg.targets
    key = "cfg3_heston" if cfg.name.startswith("cfg5") else cfg.name
    p = targets_path(key)
    if os.path.exists(p):
        with open(p) as f:
            cfg.targets = json.load(f)["targets"]
    return cfg.targets
