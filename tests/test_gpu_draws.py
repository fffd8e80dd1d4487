"""Caller-supplied draws: the reference's PathDrawSource overloads on the GPU.

ltg_gradient_of_G_draws / ltg_estimate_means_draws stand in for
gradient_of_G(kernel, params, targets, src, cfg) (expectation.hpp:300-344),
its SampleSpace overload (:354-367) and estimate_means(kernel, params, src,
paths) (:274-279) with a BufferDrawSource (rng.hpp:140-167). Checked here:
  * the draws of PhiloxNormalSource, materialised and passed back as a buffer,
    give the SAME report bit for bit as the engine's own Philox call (same
    per-path arithmetic, same chunk order);
  * arbitrary draws (heavy-tailed, scaled, exact zeros) match the reference's
    BufferDrawSource / SampleSpace calls within the 1e-10 bar, incl.
    fresh_step2_paths reading rows [P, 2P);
  * the reference's validation: dimension mismatch and too few rows raise.
"""
import numpy as np
import pytest

from paper_1901_04200_b200 import configs
from paper_1901_04200_b200.engine import Engine
from paper_1901_04200_b200.model import (BufferDrawSource, MCConfig, SampleSpace,
                                         load_model_spec)

from test_gpu_parity import assert_report_close, rel_err

pytestmark = pytest.mark.gpu


def _bits(a):
    return np.asarray(a, dtype=np.float64).view(np.uint64)


def _same_report(a, b):
    for k in ("means", "lambda_", "grad"):
        assert np.array_equal(_bits(getattr(a, k)), _bits(getattr(b, k))), k
    assert _bits([a.G])[0] == _bits([b.G])[0]


def _case(name, golden_dir):
    if name == "heston_small":
        spec = load_model_spec(f"{golden_dir}/heston_small.json")
        eng = Engine(spec)
        return spec, eng, eng.pack_params(), spec.mc.seed
    c = configs.ALL[name]()
    return c.spec, Engine(c.spec), np.asarray(c.x), c.seed


@pytest.mark.parametrize("name,paths,fresh", [("heston_small", 3001, False),
                                              ("heston_small", 1000, True),
                                              ("cfg2", 1 << 12, False),
                                              ("cfg3", 1000, False),
                                              ("cfg4", 2048 + 5, False),
                                              ("cfg4", 1000, True)])
def test_materialised_philox_equals_engine_philox(golden_dir, name, paths, fresh):
    spec, eng, x, seed = _case(name, golden_dir)
    rows = 2 * paths if fresh else paths
    src = BufferDrawSource.materialize(
        lambda p0, n: eng.fill_normals(seed, eng.N, False, p0, n), eng.N, rows)
    cfg = MCConfig(paths=paths, seed=seed, fresh_step2_paths=fresh)
    base = eng.estimate_means(x, MCConfig(paths=paths, seed=seed))
    targets = 0.9 * np.asarray(base.means)
    want = eng.gradient_of_G(x, targets, cfg, std_errors=True)
    got = eng.gradient_of_G(x, targets, cfg, std_errors=True, source=src)
    _same_report(got, want)
    assert np.array_equal(_bits(got.std_errors), _bits(want.std_errors))
    assert got.seed == seed and got.paths == paths
    m = eng.estimate_means(x, None, source=src, paths=paths)
    assert np.array_equal(_bits(m.means), _bits(base.means))
    assert np.array_equal(_bits(m.std_errors), _bits(base.std_errors))


def _odd_draws(rng, rows, dim):
    # heavy tails, a scaled block and exact zeros: not normals, still finite paths
    z = rng.standard_t(4, size=(rows, dim)) * 0.8
    z[::7] *= 1.5
    z[3, :] = 0.0
    return z


@pytest.mark.parametrize("name,paths,fresh", [("heston_small", 2000, False),
                                              ("heston_small", 700, True),
                                              ("cfg2", 1500, False),
                                              ("cfg3", 600, True),
                                              ("cfg4", 900, False)])
def test_buffer_source_vs_reference(ref, golden_dir, name, paths, fresh):
    spec, eng, x, _ = _case(name, golden_dir)
    prog = ref.program(spec)
    rng = np.random.default_rng(sum(map(ord, name)) * 7 + paths)
    z = _odd_draws(rng, 2 * paths if fresh else paths + 11, prog.N)  # spare rows are unused
    means, _ = prog.estimate_means_buffer(x, z, paths, workers=8)
    targets = means * 0.95 + 0.01
    orc = prog.gradient_of_G_buffer(x, targets, z, paths, fresh=fresh, workers=8)
    rep = eng.gradient_of_G(x, targets, MCConfig(paths=paths, seed=123, fresh_step2_paths=fresh),
                            source=BufferDrawSource(z, prog.N))
    assert_report_close(rep, orc)
    assert rep.seed == 123  # echoed, as the reference does
    m = eng.estimate_means(x, None, source=BufferDrawSource(z, prog.N), paths=paths)
    assert rel_err(m.means, means) <= 1e-10


def test_sample_space_overload(ref, golden_dir):
    spec, eng, x, _ = _case("heston_small", golden_dir)
    prog = ref.program(spec)
    rng = np.random.default_rng(5)
    n = 777
    z = rng.standard_normal((n, prog.N))
    space = SampleSpace(scenarios=n, num_randoms=prog.N, draws=z.ravel().tolist())
    means, _ = prog.estimate_means_buffer(x, z, n)
    targets = 0.8 * means
    orc = prog.gradient_of_G_space(x, targets, z, lane_width=1)
    rep = eng.gradient_of_G(x, targets, space)
    assert_report_close(rep, orc)
    assert rep.seed == 0 and rep.paths == n and rep.mode == "recompute"
    m = eng.estimate_means(x, space)
    assert rel_err(m.means, means) <= 1e-10


def test_draws_validation(golden_dir):
    spec, eng, x, seed = _case("heston_small", golden_dir)
    t = np.zeros(eng.m)
    z = np.zeros((100, eng.N))
    with pytest.raises(ValueError, match="dimension"):
        eng.gradient_of_G(x, t, MCConfig(paths=10), source=BufferDrawSource(z[:, :-2], eng.N - 2))
    with pytest.raises(ValueError, match="out of range"):
        eng.gradient_of_G(x, t, MCConfig(paths=101), source=BufferDrawSource(z, eng.N))
    with pytest.raises(ValueError, match="out of range"):
        eng.gradient_of_G(x, t, MCConfig(paths=51, fresh_step2_paths=True),
                          source=BufferDrawSource(z, eng.N))
    with pytest.raises(ValueError, match="fp64"):
        eng.gradient_of_G(x, t, MCConfig(paths=10, precision=1), source=BufferDrawSource(z, eng.N))
    # the context is still usable, and Philox calls after a draws call are unchanged
    a = eng.gradient_of_G(x, t, MCConfig(paths=500, seed=seed))
    eng.gradient_of_G(x, t, MCConfig(paths=100), source=BufferDrawSource(z, eng.N))
    b = eng.gradient_of_G(x, t, MCConfig(paths=500, seed=seed))
    _same_report(a, b)


def test_draws_on_multi_member_context(golden_dir, monkeypatch):
    # two member contexts on one GPU (the loopback collective): each member
    # uploads its own shard's rows; the report equals one context's bit for bit
    spec = load_model_spec(f"{golden_dir}/heston_small.json")
    one = Engine(spec)
    monkeypatch.setenv("LTG_LOOPBACK", "1")
    grp = Engine(spec, devices=[0, 0])
    monkeypatch.delenv("LTG_LOOPBACK")
    x = one.pack_params()
    paths = 70000
    src = BufferDrawSource(np.random.default_rng(9).standard_normal((2 * paths, one.N)), one.N)
    t = np.full(one.m, 3.0)
    for fresh in (False, True):
        cfg = MCConfig(paths=paths, seed=1, fresh_step2_paths=fresh)
        _same_report(grp.gradient_of_G(x, t, cfg, source=src),
                     one.gradient_of_G(x, t, cfg, source=src))
