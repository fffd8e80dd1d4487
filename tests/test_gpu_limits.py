"""The engine's size limits, at the limit and one past it (include/lanetape_b200.h,
engine.cpp ltg_create_heston / ltg_create_basket): 256 instruments, 8 s-nodes,
1024 leverage cells, 16 basket assets. At the limit the gradient matches the
reference (oracle/_ref) within the 1e-10 bar; one past it the context is
refused with LTG_EINVAL, before any device work (the reference itself has no
such limits — these are the device build's, stated in the header)."""
import numpy as np
import pytest

from paper_1901_04200_b200 import configs
from paper_1901_04200_b200.engine import Engine
from paper_1901_04200_b200.model import (CALL, PUT, BasketSpec, HestonParams, Instrument,
                                         LeverageGrid, McSettings, MCConfig, ModelSpec)

from test_gpu_parity import assert_report_close

pytestmark = pytest.mark.gpu


def _heston(rows, cols, n_inst, steps=96, dt=1.0 / 96):
    g = np.random.default_rng(rows * 1000 + cols * 10 + n_inst)
    t_nodes = [i * steps * dt / rows for i in range(rows)]
    s_nodes = [60.0 + 80.0 * j / max(1, cols - 1) for j in range(cols)] if cols > 1 else [0.0]
    lev = [float(v) for v in g.uniform(0.7, 1.3, rows * cols)]
    ins = [Instrument(CALL if i % 3 else PUT, float(g.uniform(80.0, 120.0)),
                      int(g.integers(1, steps + 1))) for i in range(n_inst)]
    hp = HestonParams(mu=0.01, kappa=1.5, theta=0.04, xi=0.3, rho=-0.6, v0=0.04, s0=100.0)
    return ModelSpec(hp, LeverageGrid(t_nodes, s_nodes, lev), ins, McSettings(1, steps, dt, 7))


def _check(ref, spec, paths=777, seed=3):
    eng = Engine(spec)
    x = eng.pack_params()
    t = [5.0] * eng.m
    orc = ref.program(spec).gradient_of_G(x, t, paths, seed, workers=8)
    assert_report_close(eng.gradient_of_G(x, t, MCConfig(paths=paths, seed=seed)), orc)


def test_max_instruments(ref):
    _check(ref, _heston(2, 3, 256))
    with pytest.raises(ValueError, match="256 instruments"):
        Engine(_heston(2, 3, 257))


def test_max_s_nodes(ref):
    _check(ref, _heston(3, 8, 12))
    with pytest.raises(ValueError, match="8 s-nodes"):
        Engine(_heston(3, 9, 12))


def test_max_leverage_cells(ref):
    # 128 time rows x 8 columns = 1024 cells over 256 steps
    _check(ref, _heston(128, 8, 16, steps=256, dt=1.0 / 256), paths=300)
    with pytest.raises(ValueError, match="1024 leverage cells"):
        Engine(_heston(129, 8, 16, steps=258, dt=1.0 / 258))


def test_max_basket_assets(ref):
    c = configs.cfg4()  # 16 assets: the limit (test_gpu_baseline_sizes runs it at 2^22)
    eng = Engine(c.spec)
    orc = ref.program(c.spec).gradient_of_G(c.x, c.targets, 1000, 5, workers=8)
    assert_report_close(eng.gradient_of_G(c.x, c.targets, MCConfig(paths=1000, seed=5)), orc)
    n = 17
    corr = configs.basket_correlation(n, seed=99)
    L = configs.cholesky(corr)
    spec = BasketSpec([100.0] * n, 0.02, [L[i][j] for i in range(n) for j in range(n)], [0.2] * n,
                      [Instrument(CALL, 100.0, 4)], [0], 4, 0.25)
    with pytest.raises(ValueError, match="n_assets"):
        Engine(spec)
