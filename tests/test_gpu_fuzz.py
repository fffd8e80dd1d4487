"""Randomised models against the reference (oracle/_ref), on the GPU.

The BASELINE configs pin five fixed models; these cases draw the model
itself from a seeded generator — Heston parameters on both sides of the
Feller condition, leverage grids of 1-4 rows x 1-8 columns (the grid-lookup
kernels, LEV = 1 / 2 / 4 / 8), 1-48 steps, 1-24 calls and puts at arbitrary
maturities, ragged path counts, antithetic and fresh-path options; and
correlated baskets of 1-16 assets. Per case:
  * per-path payoffs of 64 paths bit-identical to the reference tape
    (path_adjoint) on its own PhiloxNormalSource draws (Heston);
  * estimate_means (means and standard errors) and gradient_of_G within the
    1e-10 bar of test_gpu_parity.py;
  * a second call bitwise identical to the first, and the same call on the
    materialised draws (ltg_gradient_of_G_draws) bitwise identical too;
  * every 4th case: 2-5 loopback ranks on this GPU equal to one context;
  * tangent mode within the same bar where it applies (one column, <= 4 rows).
Every 8th Heston case sits on an edge of the domain (V == 0, |rho| -> 1,
heavy truncation, constant variance, a few hundred steps).
"""
import numpy as np
import pytest

from paper_1901_04200_b200 import configs
from paper_1901_04200_b200.engine import Engine
from paper_1901_04200_b200.model import (CALL, PUT, BasketSpec, BufferDrawSource, HestonParams,
                                         Instrument, LeverageGrid, McSettings, MCConfig,
                                         ModelSpec)

from test_gpu_parity import TOL, assert_report_close, rel_err

pytestmark = pytest.mark.gpu


def random_heston(seed):
    g = np.random.default_rng(seed)
    s0 = float(g.uniform(50.0, 150.0))
    hp = HestonParams(mu=float(g.uniform(-0.05, 0.05)), kappa=float(g.uniform(0.0, 3.0)),
                      theta=float(g.uniform(0.01, 0.1)), xi=float(g.uniform(0.0, 1.2)),
                      rho=float(g.uniform(-0.95, 0.95)), v0=float(g.uniform(0.005, 0.1)), s0=s0)
    edge = seed % 8  # every 8th family member takes an edge of the model's domain
    if edge == 0:
        hp.v0, hp.theta = 0.0, 0.0                # V == 0 throughout: the sqrt-at-0 branch
    elif edge == 1:
        hp.rho = float(g.choice([-0.999, 0.999]))  # rho_comp near 0
    elif edge == 2:
        hp.xi = 2.5                               # variance truncated on most steps
    elif edge == 3:
        hp.kappa, hp.xi = 0.0, 0.0                # V == v0: local-vol-only paths
    steps = int(g.integers(1, 49)) if edge != 4 else int(g.integers(100, 300))
    dt = float(1.0 / g.choice([12, 52, 252, 365]))
    rows, cols = int(g.integers(1, 5)), int(g.choice([1, 2, 3, 5, 8]))
    t_nodes = [0.0] + sorted(set(float(v) for v in g.uniform(0.0, steps * dt, rows - 1)))
    s_nodes = sorted(set(float(v) for v in g.uniform(0.6 * s0, 1.4 * s0, cols)))
    lev = [float(v) for v in g.uniform(0.5, 1.5, len(t_nodes) * len(s_nodes))]
    m = int(g.integers(1, 25))
    ins = [Instrument(int(g.choice([CALL, PUT])), float(s0 * g.uniform(0.7, 1.3)),
                      int(g.integers(1, steps + 1))) for _ in range(m)]
    spec = ModelSpec(hp, LeverageGrid(t_nodes, s_nodes, lev), ins,
                     McSettings(1, steps, dt, int(g.integers(0, 2**63))))
    opts = dict(paths=int(g.integers(1, 6000)), seed=int(g.integers(0, 2**64, dtype=np.uint64)),
                antithetic=bool(g.integers(0, 2)), fresh=bool(g.integers(0, 4) == 0))
    return spec, opts, g


def random_basket(seed):
    g = np.random.default_rng(seed)
    n = int(g.integers(1, 17))
    L = configs.cholesky(configs.basket_correlation(n, seed=seed))
    steps = int(g.integers(1, 61))
    ins, assets = [], []
    for _ in range(int(g.integers(1, 25))):
        a = int(g.integers(0, n))
        ins.append(Instrument(int(g.choice([CALL, PUT])), float(g.uniform(70.0, 130.0)),
                              int(g.integers(1, steps + 1))))
        assets.append(a)
    spec = BasketSpec([float(v) for v in g.uniform(80.0, 120.0, n)], float(g.uniform(-0.02, 0.05)),
                      [L[i][j] for i in range(n) for j in range(n)],
                      [0.2] * n, ins, assets, steps, float(1.0 / g.choice([12, 50, 252])))
    x = [float(v) for v in g.uniform(0.1, 0.5, n)]
    opts = dict(paths=int(g.integers(1, 6000)), seed=int(g.integers(0, 2**64, dtype=np.uint64)),
                antithetic=bool(g.integers(0, 2)), fresh=bool(g.integers(0, 4) == 0))
    return spec, x, opts, g


def _check(ref, spec, x, opts, g, tangent_ok):
    eng = Engine(spec)
    prog = ref.program(spec)
    P, seed, anti, fresh = opts["paths"], opts["seed"], opts["antithetic"], opts["fresh"]
    means, se = prog.estimate_means(x, P, seed, antithetic=anti, workers=8)
    res = eng.estimate_means(x, MCConfig(paths=P, seed=seed, antithetic=anti))
    assert rel_err(res.means, means) <= TOL
    if P > 1:
        # standard errors compared as sample variances, with a floor at the
        # rounding noise of sum(y^2) - P mean^2 (degenerate, zero-variance
        # payoffs leave only that noise, summed in different orders)
        va, vb = np.asarray(res.std_errors) ** 2 * P, np.asarray(se) ** 2 * P
        ey2 = np.asarray(means) ** 2 + np.maximum(va, vb)
        assert np.all(np.abs(va - vb) <= 1e-8 * np.maximum(va, vb) + 1e-12 * ey2)
    targets = means * g.uniform(0.8, 1.2, len(means)) + g.uniform(-0.5, 0.5, len(means))
    orc = prog.gradient_of_G(x, targets, P, seed, antithetic=anti, fresh=fresh, workers=8)
    cfg = MCConfig(paths=P, seed=seed, antithetic=anti, fresh_step2_paths=fresh)
    rep = eng.gradient_of_G(x, targets, cfg)
    assert_report_close(rep, orc)
    again = eng.gradient_of_G(x, targets, cfg)
    assert again.G == rep.G and again.grad == rep.grad and again.means == rep.means
    # the same paths as caller draws (the materialised PhiloxNormalSource,
    # antithetic pairs included, through the DRAWS kernels): the same report
    rows = 2 * P if fresh else P
    src = BufferDrawSource(eng.fill_normals(seed, eng.N, anti, 0, rows), eng.N)
    viad = eng.gradient_of_G(x, targets, MCConfig(paths=P, seed=seed, fresh_step2_paths=fresh),
                             source=src)
    assert viad.G == rep.G and viad.grad == rep.grad and viad.means == rep.means
    if tangent_ok:
        t = eng.gradient_of_G(x, targets, cfg, method="tangent")
        assert_report_close(t, orc)
    return eng, prog


@pytest.mark.parametrize("case", range(64))
def test_random_heston_models(ref, case):
    spec, opts, g = random_heston(1000 + case)
    tangent_ok = spec.grid.cols() == 1 and spec.grid.rows() <= 4
    x = ref.program(spec).initial_params()
    eng, prog = _check(ref, spec, x, opts, g, tangent_ok)
    # per-path payoffs, bit for bit, against the reference tape on its own draws
    n, path0 = 64, int(g.integers(0, 1 << 40))
    y = eng.path_payoffs(x, opts["seed"], opts["antithetic"], path0, n)
    z = ref.fill_normals(opts["seed"], prog.N, opts["antithetic"], path0, n)
    want = np.stack([prog.path_adjoint(x, z[i])[0] for i in range(n)])
    assert np.array_equal(y.view(np.uint64), want.view(np.uint64))
    if case % 4 == 0:
        _check_ranks(spec, x, opts, g)


def _check_ranks(spec, x, opts, g):
    # W loopback ranks on this GPU (test_gpu_parity.py::test_multi_rank_paths_on_one_gpu),
    # W = 2..5, possibly more ranks than chunks: reports equal to one context's, bit for bit
    import os
    world = int(g.integers(2, 6))
    os.environ["LTG_LOOPBACK"] = "1"
    try:
        grp = Engine(spec, devices=[0] * world)
    finally:
        os.environ.pop("LTG_LOOPBACK")
    t = [1.0] * grp.m
    cfg = MCConfig(paths=opts["paths"], seed=opts["seed"], antithetic=opts["antithetic"],
                   fresh_step2_paths=opts["fresh"])
    assert grp.gradient_of_G(x, t, cfg).to_json() == Engine(spec).gradient_of_G(x, t, cfg).to_json()


@pytest.mark.parametrize("case", range(16))
def test_random_baskets(ref, case):
    spec, x, opts, g = random_basket(2000 + case)
    _check(ref, spec, x, opts, g, False)
    if case % 4 == 0:
        _check_ranks(spec, x, opts, g)
