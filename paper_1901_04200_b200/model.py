"""Model and configuration types, mirroring the reference's model layer.

Python mirror of ``lanetape``'s ``HestonParams``/``LeverageGrid``/``Instrument``/
``McSettings``/``ModelSpec`` (heston.hpp:20-114), their validation
(heston.hpp:30-130), JSON I/O with the reference's key layout
(heston.hpp:132-210) and ``pack_params``/``unpack_params`` (heston.hpp:212-232);
plus ``MCConfig``/``GradientReport``/``MeansResult`` (expectation.hpp:25-82).
These are plain host-side descriptions: the CUDA engine receives them through
the C ABI in ``include/lanetape_b200.h``.
"""
from __future__ import annotations

import bisect
import json
import math
from dataclasses import dataclass, field
from typing import List, Optional, Sequence

CALL, PUT = 0, 1
HESTON_FREE_PARAMS = 5  # heston.hpp:213


@dataclass
class HestonParams:
    mu: float = 0.0
    kappa: float = 1.0
    theta: float = 0.04
    xi: float = 0.5
    rho: float = -0.7
    v0: float = 0.04
    s0: float = 100.0


def validate_params(p: HestonParams) -> None:
    """heston.hpp:30-41"""
    def bad(what):
        raise ValueError("HestonParams: " + what)
    if not (p.s0 > 0.0):
        bad("s0 must be > 0")
    if not (p.v0 >= 0.0):
        bad("v0 must be >= 0")
    if not (p.theta >= 0.0):
        bad("theta must be >= 0")
    if not (p.kappa >= 0.0):
        bad("kappa must be >= 0")
    if not (p.xi >= 0.0):
        bad("xi must be >= 0")
    if not (abs(p.rho) < 1.0):
        bad("rho must satisfy |rho| < 1")
    if not math.isfinite(p.mu):
        bad("mu must be finite")


@dataclass
class LeverageGrid:
    t_nodes: List[float] = field(default_factory=lambda: [0.0])
    s_nodes: List[float] = field(default_factory=lambda: [0.0])
    values: List[float] = field(default_factory=lambda: [1.0])  # t-major

    def rows(self) -> int:
        return len(self.t_nodes)

    def cols(self) -> int:
        return len(self.s_nodes)

    def at(self, row: int, col: int) -> float:
        return self.values[row * self.cols() + col]


def validate_grid(g: LeverageGrid) -> None:
    """heston.hpp:57-70"""
    def bad(what):
        raise ValueError("LeverageGrid: " + what)
    if not g.t_nodes or not g.s_nodes:
        bad("node lists must be non-empty")
    for i in range(1, len(g.t_nodes)):
        if not (g.t_nodes[i] > g.t_nodes[i - 1]):
            bad("t_nodes must be strictly ascending")
    for i in range(1, len(g.s_nodes)):
        if not (g.s_nodes[i] > g.s_nodes[i - 1]):
            bad("s_nodes must be strictly ascending")
    if len(g.values) != len(g.t_nodes) * len(g.s_nodes):
        bad("values must hold t_nodes x s_nodes entries")
    for v in g.values:
        if not math.isfinite(v) or v < 0.0:
            bad("values must be finite and >= 0")


def floor_index(nodes: Sequence[float], x: float) -> int:
    """heston.hpp:72-76: largest i with nodes[i] <= x, clamped to 0."""
    i = bisect.bisect_right(list(nodes), x)
    return 0 if i == 0 else i - 1


@dataclass
class Instrument:
    kind: int = CALL
    strike: float = 100.0
    maturity_step: int = 1


@dataclass
class McSettings:
    paths: int = 0
    steps: int = 0
    dt: float = 0.0
    seed: int = 0


@dataclass
class ModelSpec:
    heston: HestonParams = field(default_factory=HestonParams)
    grid: LeverageGrid = field(default_factory=LeverageGrid)
    instruments: List[Instrument] = field(default_factory=list)
    mc: McSettings = field(default_factory=McSettings)


def validate_spec(s: ModelSpec, check_paths: bool = True) -> None:
    """heston.hpp:116-130"""
    validate_params(s.heston)
    validate_grid(s.grid)
    if check_paths and s.mc.paths == 0:
        raise ValueError("mc: paths must be > 0")
    if s.mc.steps == 0:
        raise ValueError("mc: steps must be > 0")
    if not (s.mc.dt > 0.0):
        raise ValueError("mc: dt must be > 0")
    if not s.instruments:
        raise ValueError("instruments: list must be non-empty")
    for i, ins in enumerate(s.instruments):
        if not (ins.strike > 0.0):
            raise ValueError(f"instruments[{i}]: strike must be > 0")
        if ins.maturity_step == 0 or ins.maturity_step > s.mc.steps:
            raise ValueError(f"instruments[{i}]: maturity_step must be in [1, steps]")


def model_spec_from_json(j: dict) -> ModelSpec:
    """heston.hpp:132-175 (same keys; rows of grid.values are t-major)."""
    h = j["heston"]
    s = ModelSpec()
    s.heston = HestonParams(mu=float(h["mu"]), kappa=float(h["kappa"]), theta=float(h["theta"]),
                            xi=float(h["xi"]), rho=float(h["rho"]), v0=float(h["v0"]),
                            s0=float(h["s0"]))
    g = j["grid"]
    vals: List[float] = []
    for row in g["values"]:
        if len(row) != len(g["s_nodes"]):
            raise ValueError("grid: every values row needs one entry per s_node")
        vals.extend(float(v) for v in row)
    s.grid = LeverageGrid([float(t) for t in g["t_nodes"]], [float(v) for v in g["s_nodes"]], vals)
    for ji in j["instruments"]:
        kind = ji["kind"]
        if kind not in ("call", "put"):
            raise ValueError('instruments: kind must be "call" or "put"')
        s.instruments.append(Instrument(CALL if kind == "call" else PUT, float(ji["strike"]),
                                        int(ji["maturity_step"])))
    mc = j["mc"]
    s.mc = McSettings(int(mc["paths"]), int(mc["steps"]), float(mc["dt"]), int(mc["seed"]))
    validate_spec(s)
    return s


def to_json(s: ModelSpec) -> dict:
    """heston.hpp:177-202 (key order pinned)."""
    cols = s.grid.cols()
    return {
        "heston": {"kappa": s.heston.kappa, "theta": s.heston.theta, "xi": s.heston.xi,
                   "rho": s.heston.rho, "v0": s.heston.v0, "s0": s.heston.s0, "mu": s.heston.mu},
        "grid": {"t_nodes": list(s.grid.t_nodes), "s_nodes": list(s.grid.s_nodes),
                 "values": [list(s.grid.values[r * cols:(r + 1) * cols])
                            for r in range(s.grid.rows())]},
        "instruments": [{"kind": "call" if i.kind == CALL else "put", "strike": i.strike,
                         "maturity_step": i.maturity_step} for i in s.instruments],
        "mc": {"paths": s.mc.paths, "steps": s.mc.steps, "dt": s.mc.dt, "seed": s.mc.seed},
    }


def load_model_spec(path: str) -> ModelSpec:
    """heston.hpp:204-210"""
    with open(path) as f:
        return model_spec_from_json(json.load(f))


def pack_params(p: HestonParams, g: LeverageGrid) -> List[float]:
    """heston.hpp:212-219: [kappa, theta, xi, rho, v0, L row-major]."""
    return [p.kappa, p.theta, p.xi, p.rho, p.v0] + list(g.values)


def unpack_params(x: Sequence[float], p: HestonParams, g: LeverageGrid) -> None:
    """heston.hpp:221-232"""
    if len(x) != HESTON_FREE_PARAMS + len(g.values):
        raise ValueError("unpack_params: packed size mismatch")
    p.kappa, p.theta, p.xi, p.rho, p.v0 = (float(v) for v in x[:5])
    g.values = [float(v) for v in x[5:]]


@dataclass
class BasketSpec:
    """Config-4 correlated log-Euler GBM basket (no reference model-layer
    counterpart; its oracle program is recorded in oracle/ref_driver.cpp)."""
    s0: List[float]
    r: float
    chol: List[float]            # n*n lower-triangular, row-major
    sigma: List[float]           # recorded-at vols (the parameters)
    instruments: List[Instrument]
    inst_asset: List[int]
    steps: int
    dt: float

    @property
    def n_assets(self) -> int:
        return len(self.s0)


# ---- expectation.hpp ----------------------------------------------------

MODE_RECOMPUTE, MODE_STORE = 0, 1
FP64, FP32 = 0, 1


@dataclass
class MCConfig:
    """expectation.hpp:25-39. lane_width / worker_threads / store_limit_bytes
    steer the CPU reference only; accepted and ignored by the GPU engine."""
    paths: int = 0
    seed: int = 0
    antithetic: bool = False
    lane_width: int = 4
    worker_threads: int = 1
    memory_mode: int = MODE_RECOMPUTE
    fresh_step2_paths: bool = False
    store_limit_bytes: int = 3 << 30
    precision: int = FP64


@dataclass
class SampleSpace:
    """expectation.hpp:46-54: an explicit, uniformly weighted scenario set
    (scenario-major draws, scenarios * num_randoms)."""
    scenarios: int = 0
    num_randoms: int = 0
    draws: Sequence[float] = field(default_factory=list)

    def row(self, s: int) -> Sequence[float]:
        return self.draws[s * self.num_randoms:(s + 1) * self.num_randoms]


class BufferDrawSource:
    """rng.hpp:140-167: draws read from a flat path-major buffer (row p = the
    `dimension` draws of path p)."""

    def __init__(self, draws, dimension: int):
        import numpy as np
        self.draws = np.ascontiguousarray(draws, dtype=np.float64).ravel()
        self.dim = int(dimension)
        if self.dim == 0 or self.draws.size % self.dim != 0:
            raise ValueError("BufferDrawSource: buffer size not a multiple of dimension")

    @staticmethod
    def materialize(fill, dimension: int, paths: int) -> "BufferDrawSource":
        """rng.hpp:149-154 for a source given as fill(path0, npaths) -> the
        path-major draws of paths [path0, path0 + npaths), e.g.
        ``lambda p0, n: engine.fill_normals(seed, dim, anti, p0, n)``."""
        return BufferDrawSource(fill(0, paths), dimension)

    def dimension(self) -> int:
        return self.dim

    def paths(self) -> int:
        return self.draws.size // self.dim

    def fill(self, path: int):
        if path >= self.paths():
            raise IndexError("BufferDrawSource: path index out of range")
        return self.draws[path * self.dim:(path + 1) * self.dim]


def memory_mode_name(m: int) -> str:
    """expectation.hpp:19-21"""
    return "store" if m == MODE_STORE else "recompute"


@dataclass
class MeansResult:
    means: List[float]
    std_errors: List[float]
    paths: int


@dataclass
class GradientReport:
    G: float
    means: List[float]
    lambda_: List[float]
    grad: List[float]
    paths: int
    mode: str
    seed: int

    def to_json(self, indent: Optional[int] = 2) -> str:
        """expectation.hpp:71-81, pinned key order G, means, lambda, grad, paths, mode, seed."""
        d = {"G": self.G, "means": self.means, "lambda": self.lambda_, "grad": self.grad,
             "paths": self.paths, "mode": self.mode, "seed": self.seed}
        return json.dumps(d, indent=indent)
