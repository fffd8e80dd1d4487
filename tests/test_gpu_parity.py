"""GPU parity: the CUDA engine (through the C ABI) against the CPU oracle.

The oracle is the reference library itself compiled in place
(oracle/_ref/libltref.so) — its gradient_of_G / estimate_means /
PhiloxNormalSource — on the same seeded inputs. Bars (north_star,
BASELINE.json):
  * random draws: bit-exact;
  * E[y], lambda, G, grad: relative error <= 1e-10 in fp64 with the
    denominator max(|a|, |b|, floor), floor = 1e-12 * max|vector|
    (tests/support/oracles.hpp:19-22 style rel_err).
"""
import math
import os

import numpy as np
import pytest

from paper_1901_04200_b200 import configs
from paper_1901_04200_b200.engine import Engine, EvalError
from paper_1901_04200_b200.model import MCConfig, MODE_STORE, load_model_spec

pytestmark = pytest.mark.gpu

TOL = 1e-10


def rel_err(a, b, floor_frac=1e-12):
    a, b = np.asarray(a, dtype=float), np.asarray(b, dtype=float)
    floor = floor_frac * max(np.max(np.abs(a)), np.max(np.abs(b)), 1e-300)
    return np.max(np.abs(a - b) / np.maximum(np.maximum(np.abs(a), np.abs(b)), floor))


def assert_report_close(rep, orc, tol=TOL):
    assert rel_err(rep.means, orc["means"]) <= tol, (rep.means, orc["means"])
    assert rel_err(rep.lambda_, orc["lambda_"]) <= tol
    assert rel_err([rep.G], [orc["G"]]) <= tol, (rep.G, orc["G"])
    assert rel_err(rep.grad, orc["grad"]) <= tol, (np.asarray(rep.grad), orc["grad"])


@pytest.fixture(scope="module")
def small(golden_dir):
    spec = load_model_spec(f"{golden_dir}/heston_small.json")
    return spec, Engine(spec)


# ---------------------------------------------------------------- RNG ----

@pytest.mark.parametrize("seed,dim,anti,path0", [
    (42, 8, False, 7),                   # test_rng.cpp:67-74 hand-derived draws
    (20190114, 1512, False, 0),          # config-3 path dimension
    (9001, 6, False, 123456789),
    (5, 3, False, 0),                    # odd dimension (rng.hpp:124)
    (77, 4, True, 0),                    # antithetic pairing (rng.hpp:114-115)
    (31415, 33, True, (1 << 40) + 3),    # high path word, odd dim, antithetic
    ((1 << 63) + 12345, 128, False, (1 << 33) + 17),
])
def test_normals_bit_exact(ref, small, seed, dim, anti, path0):
    eng = small[1]
    npaths = 300
    g = eng.fill_normals(seed, dim, anti, path0, npaths)
    r = ref.fill_normals(seed, dim, anti, path0, npaths)
    mism = int(np.sum(g.view(np.uint64) != r.view(np.uint64)))
    assert mism == 0, f"{mism} of {g.size} draws differ"


def test_hand_derived_draws(small):
    z = small[1].fill_normals(42, 8, False, 7, 1)[0]
    assert z[6] == 0.020415871554285415
    assert z[7] == -0.17620946540988347


def test_rng_uses_validated_libm_log(small):
    assert small[1].rng_exact


def test_normals_bulk_tail_exact(ref, small):
    # 2^16 paths x 64 draws: ~630k tail draws through the glibc-log restatement
    g = small[1].fill_normals(2718, 64, False, 1 << 20, 1 << 16)
    r = ref.fill_normals(2718, 64, False, 1 << 20, 1 << 16)
    assert np.array_equal(g.view(np.uint64), r.view(np.uint64))


def _gen_uniform(k):
    """The generator's uniforms: (2k+1)*2^-53, k a 52-bit integer (rng.hpp:38-40)."""
    return (2.0 * np.asarray(k, dtype=np.float64) + 1.0) * 2.0 ** -53


def test_inverse_normal_all_rows_bit_exact(ref, small):
    # every AS241 row on the device, including the r > 5 row that Philox
    # practically never reaches (p < 1.4e-11) and the generator's endpoints
    # 2^-53 / 1 - 2^-53 (test_rng.cpp:38-45)
    top = (1 << 52) - 1
    rng = np.random.default_rng(1901)
    ks = [0, 1, 2, 3, top, top - 1, top - 7, 1 << 51, (1 << 51) - 1]
    for p in (1e-300, 1e-16, 1e-12, 1.388e-11, 1.389e-11, 1e-10, 1e-6, 0.0749999, 0.0750001,
              0.3, 0.5):
        k = int(p * 2.0 ** 52)
        ks += [k, k + 1, top - k, top - k - 1]
    ks += list(rng.integers(0, 1 << 52, 20000))  # mixed central / tail
    ks += list(rng.integers(0, 1 << 28, 2000))   # deep lower tail (r > 5 included)
    ks += list(top - rng.integers(0, 1 << 28, 2000))
    p = _gen_uniform(np.clip(np.asarray(ks, dtype=np.int64), 0, top))
    z = small[1].inverse_normal(p)
    r = np.array([ref.inverse_normal_cdf(float(v)) for v in p])
    assert np.sum(np.minimum(p, 1 - p) < 1.38e-11) > 10  # the r > 5 row was exercised
    mism = np.flatnonzero(z.view(np.uint64) != r.view(np.uint64))
    assert mism.size == 0, [(p[i], z[i], r[i]) for i in mism[:5]]


def test_inverse_normal_domain(small):
    with pytest.raises(ValueError):
        small[1].inverse_normal([0.5, 0.0])
    with pytest.raises(ValueError):
        small[1].inverse_normal([1.0])


@pytest.mark.parametrize("name", ["heston_small", "cfg1", "cfg2", "cfg3", "cfg4"])
def test_per_path_payoffs_bit_exact(ref, golden_dir, name):
    # the GPU forward replays the reference's tape arithmetic operation for
    # operation (glibc exp and log included): per-path outputs are identical
    if name == "heston_small":
        spec = load_model_spec(f"{golden_dir}/heston_small.json")
        x = None
    else:
        c = configs.ALL[name]()
        spec, x = c.spec, c.x
    eng = Engine(spec)
    prog = ref.program(spec)
    if x is None:
        x = prog.initial_params()
    assert eng.rng_exact
    n, p0, seed = 200, 12345, 777
    y = eng.path_payoffs(x, seed, False, p0, n)
    z = ref.fill_normals(seed, prog.N, False, p0, n)
    want = np.stack([prog.path_adjoint(x, z[i])[0] for i in range(n)])
    assert np.array_equal(y.view(np.uint64), want.view(np.uint64)), \
        f"{int(np.sum(y != want))} of {y.size} payoffs differ"


# ------------------------------------------------------ two-pass gradient ----

def _targets_from(ref_prog, x, paths, seed, scale=0.9):
    means, _ = ref_prog.estimate_means(x, paths, seed, workers=8)
    return scale * means


@pytest.mark.parametrize("paths", [64, 1000, 4096 + 37])
def test_heston_small_gradient(ref, small, paths):
    spec, eng = small
    prog = ref.program(spec)
    x = prog.initial_params()
    targets = _targets_from(prog, x, paths, spec.mc.seed)
    orc = prog.gradient_of_G(x, targets, paths, spec.mc.seed, workers=8)
    rep = eng.gradient_of_G(x, targets, MCConfig(paths=paths, seed=spec.mc.seed))
    assert_report_close(rep, orc)


@pytest.mark.parametrize("name,paths", [("cfg1", 1 << 16), ("cfg2", 1 << 14), ("cfg3", 1 << 12),
                                        ("cfg3", 3000)])
def test_baseline_configs_gradient(ref, name, paths):
    c = configs.ALL[name]()
    eng = Engine(c.spec)
    prog = ref.program(c.spec)
    targets = c.targets if c.targets is not None else _targets_from(prog, c.truth, paths, 4242)
    orc = prog.gradient_of_G(c.x, targets, paths, c.seed, workers=8)
    rep = eng.gradient_of_G(c.x, targets, MCConfig(paths=paths, seed=c.seed))
    assert_report_close(rep, orc)


@pytest.mark.parametrize("paths,fresh,anti", [(1 << 12, False, False), (3001, False, False),
                                              (2048, True, False), (2049, False, True)])
def test_basket_gradient(ref, paths, fresh, anti):
    # config 4: 16 correlated GBMs; store mode (pass 1 keeps (S, W) at the
    # maturity) and, with fresh_step2_paths, recompute mode
    c = configs.cfg4()
    eng = Engine(c.spec)
    prog = ref.program(c.spec)
    orc = prog.gradient_of_G(c.x, c.targets, paths, c.seed, antithetic=anti, fresh=fresh,
                             workers=8)
    rep = eng.gradient_of_G(c.x, c.targets, MCConfig(paths=paths, seed=c.seed,
                                                      fresh_step2_paths=fresh, antithetic=anti))
    assert_report_close(rep, orc)


def test_basket_multi_maturity_puts(ref):
    # general maturities, puts and calls, fewer assets
    import math
    from paper_1901_04200_b200.model import BasketSpec, Instrument, CALL, PUT
    n, steps = 5, 12
    corr = configs.basket_correlation(n, seed=99)
    L = configs.cholesky(corr)
    ins, assets = [], []
    for a in range(n):
        ins += [Instrument(CALL, 100.0, 4 + a), Instrument(PUT, 98.0, steps)]
        assets += [a, a]
    spec = BasketSpec([100.0 + a for a in range(n)], 0.03, [L[i][j] for i in range(n)
                                                             for j in range(n)],
                      [0.2] * n, ins, assets, steps, 1.0 / 12)
    x = [0.15 + 0.05 * a for a in range(n)]
    eng = Engine(spec)
    prog = ref.program(spec)
    t = [1.0] * len(ins)
    for fresh in (False, True):
        orc = prog.gradient_of_G(x, t, 4099, 9, fresh=fresh, workers=8)
        rep = eng.gradient_of_G(x, t, MCConfig(paths=4099, seed=9, fresh_step2_paths=fresh))
        assert_report_close(rep, orc)


# fp32 mode vs the fp64 oracle on the same paths, one bar per
# BASELINE config the mode accepts (measured errors in the comments: at the
# sizes below, gpurun_out/fp32_error.log). Relative errors use the floors
# 1e-6 * max|means| and 1e-3 * max|grad|. Config 2's bar is the widest: its 40
# leverage cells include outer spot buckets that few paths visit, and an fp32
# path that lands on the other side of a bucket boundary moves that step's
# leverage adjoint to the neighbouring cell.
FP32_TOL = {"cfg1": {"means": 1e-5, "G": 1e-4, "grad": 1e-4},     # 7.5e-7 / 9.0e-6 / 1.5e-5
            "cfg2": {"means": 1e-5, "G": 1e-4, "grad": 5e-3},     # 3.3e-6 / 9.2e-6 / 1.8e-3
            "cfg3": {"means": 1e-4, "G": 1e-3, "grad": 1e-3}}     # 2.0e-5 / 1.2e-4 / 9.8e-5


@pytest.mark.parametrize("name,paths", [("cfg1", 1 << 16), ("cfg2", 1 << 14), ("cfg3", 1 << 14),
                                        ("cfg2", 1 << 20), ("cfg3", 1 << 20)])
def test_fp32_mode_against_fp64_oracle(ref, name, paths):
    # float state/adjoint and float AS241 on the same Philox words
    from paper_1901_04200_b200.model import FP32
    tol = FP32_TOL[name]
    c = configs.ALL[name]()
    t = configs.load_targets(c) or c.targets
    prog = ref.program(c.spec)
    orc = prog.gradient_of_G(c.x, t, paths, c.seed, workers=os.cpu_count())
    rep = Engine(c.spec).gradient_of_G(c.x, t, MCConfig(paths=paths, seed=c.seed, precision=FP32))
    assert rel_err(rep.means, orc["means"], 1e-6) <= tol["means"]
    assert rel_err([rep.G], [orc["G"]]) <= tol["G"]
    assert rel_err(rep.grad, orc["grad"], 1e-3) <= tol["grad"]


def test_fp32_gradient_refused_below_feller(ref, golden_dir):
    # heston_small (2*kappa*theta = 0.12 < xi^2 = 0.25): V sits at the
    # truncation kink on many paths and fp32 adjoints are off by up to 0.25
    # (measured over seeds 3-5, 2^12..2^20 paths) — the gradient is refused;
    # fp32 means still meet their bar
    from paper_1901_04200_b200.model import FP32
    spec = load_model_spec(f"{golden_dir}/heston_small.json")
    prog = ref.program(spec)
    x = prog.initial_params()
    eng = Engine(spec)
    with pytest.raises(ValueError, match="Feller"):
        eng.gradient_of_G(x, [1.0] * eng.m, MCConfig(paths=4096, seed=3, precision=FP32))
    means, _ = prog.estimate_means(x, 4096, 3, workers=8)
    r = eng.estimate_means(x, MCConfig(paths=4096, seed=3, precision=FP32))
    assert rel_err(r.means, means, 1e-6) <= 1e-4
    # at the Feller boundary itself the call is accepted
    xb = list(x)
    xb[2] = (2.0 * x[0] * x[1]) ** 0.5
    eng.gradient_of_G(xb, [1.0] * eng.m, MCConfig(paths=1024, seed=3, precision=FP32))


def test_estimate_means_and_std_errors(ref, small):
    spec, eng = small
    prog = ref.program(spec)
    x = prog.initial_params()
    means, se = prog.estimate_means(x, 5000, 99, workers=8)
    r = eng.estimate_means(x, MCConfig(paths=5000, seed=99))
    assert rel_err(r.means, means) <= TOL
    assert rel_err(r.std_errors, se) <= 1e-8  # sqrt of a cancelling difference


def test_antithetic(ref, small):
    spec, eng = small
    prog = ref.program(spec)
    x = prog.initial_params()
    t = _targets_from(prog, x, 2048, 5)
    orc = prog.gradient_of_G(x, t, 2048 + 1, 5, antithetic=True, workers=8)
    rep = eng.gradient_of_G(x, t, MCConfig(paths=2048 + 1, seed=5, antithetic=True))
    assert_report_close(rep, orc)


def test_fresh_step2_paths(ref, small):
    spec, eng = small
    prog = ref.program(spec)
    x = prog.initial_params()
    t = _targets_from(prog, x, 3000, 11)
    orc = prog.gradient_of_G(x, t, 3000, 11, fresh=True, workers=8)
    rep = eng.gradient_of_G(x, t, MCConfig(paths=3000, seed=11, fresh_step2_paths=True))
    assert_report_close(rep, orc)


@pytest.mark.parametrize("env", [{"LTG_ZSTORE": "0"}, {"LTG_ZCHUNKS_MAX": "3"},
                                 {"LTG_HBM_BUDGET_GB": "0.1"}, {"LTG_HBM_BUDGET_GB": "0"},
                                 {"LTG_CKPT_STEPS": "16"},
                                 {"LTG_CKPT_STEPS": "16", "LTG_ZSTORE": "0"},
                                 {"LTG_SAFE": "1"}])
def test_memory_plans_bitwise_identical(env):
    # pass 2 reading stored draws, regenerating them, or mixing both per
    # chunk, with 8- or 16-step checkpoints: the same arithmetic on the same
    # draws, so the report must not change by a single bit
    import os
    c = configs.cfg3()
    eng = Engine(c.spec)
    cfg = MCConfig(paths=5000, seed=c.seed)
    t = configs.load_targets(c)
    base = eng.gradient_of_G(c.x, t, cfg)
    assert eng.timing()["z_bytes"] > 0 and eng.timing()["seg_steps"] == 8
    old = {k: os.environ.get(k) for k in env}
    os.environ.update(env)
    try:
        rep = eng.gradient_of_G(c.x, t, cfg)
    finally:
        for k, v in old.items():
            if v is None:
                os.environ.pop(k)
            else:
                os.environ[k] = v
    assert rep.to_json() == base.to_json()


def test_hbm_budget_api():
    # ltg_set_hbm_budget: a tiny budget forces the no-table plan (pass 2 in
    # waves); the report does not change
    c = configs.cfg3()
    t = configs.load_targets(c)
    cfg = MCConfig(paths=5000, seed=c.seed)
    eng = Engine(c.spec)
    base = eng.gradient_of_G(c.x, t, cfg)
    assert eng.timing()["z_bytes"] > 0
    eng.set_hbm_budget(1 << 20)
    rep = eng.gradient_of_G(c.x, t, cfg)
    assert eng.timing()["z_bytes"] == 0 and eng.timing()["ckpt_bytes"] == 0
    assert rep.to_json() == base.to_json()
    eng.set_hbm_budget(0)
    eng.gradient_of_G(c.x, t, cfg)
    assert eng.timing()["z_bytes"] > 0


def test_nccl_attached_single_rank_bitwise():
    # the multi-GPU code path (run-time NCCL, in-place all-gather of the chunk
    # tables, all-reduce of the rare flag) on a one-rank communicator
    from paper_1901_04200_b200.engine import nccl_unique_id
    c = configs.cfg3()
    t = configs.load_targets(c)
    cfg = MCConfig(paths=4099, seed=c.seed)
    base = Engine(c.spec).gradient_of_G(c.x, t, cfg)
    eng = Engine(c.spec)
    eng.attach_nccl(nccl_unique_id(), 0, 1)
    assert eng.gradient_of_G(c.x, t, cfg).to_json() == base.to_json()


@pytest.mark.parametrize("fresh", [False, True])
def test_basket_safe_rerun_bitwise(fresh):
    # the basket's fast exp path (rare flag instead of the |x| >= 512 guard)
    # against the always-exact kernels, store and recompute pass 2
    import os
    c = configs.cfg4()
    eng = Engine(c.spec)
    cfg = MCConfig(paths=3001, seed=c.seed, fresh_step2_paths=fresh)
    base = eng.gradient_of_G(c.x, c.targets, cfg)
    os.environ["LTG_SAFE"] = "1"
    try:
        rep = eng.gradient_of_G(c.x, c.targets, cfg)
    finally:
        os.environ.pop("LTG_SAFE")
    assert rep.to_json() == base.to_json()


# ------------------------------------------- tangent-mode alternative ----

@pytest.mark.parametrize("name,paths,anti,fresh", [("cfg3", 4099, False, False),
                                                  ("cfg3", 2048, True, False),
                                                  ("cfg3", 3001, False, True),
                                                  ("cfg1", 1 << 14, False, False),
                                                  ("cfg1", 5000, True, True)])
def test_tangent_mode_matches_reference(ref, name, paths, anti, fresh):
    # pathwise tangents instead of pass 2: the reference's estimator on the
    # same paths (grad = sum_i lambda_i J_i / P), so the same 1e-10 bar against
    # the reference's two-pass gradient_of_G; G, means and lambda come from
    # the same forward and are pass 1's bit for bit
    c = configs.ALL[name]()
    eng = Engine(c.spec)
    prog = ref.program(c.spec)
    t = configs.load_targets(c) or _targets_from(prog, c.truth, paths, 4242)
    cfg = MCConfig(paths=paths, seed=c.seed, antithetic=anti, fresh_step2_paths=fresh)
    orc = prog.gradient_of_G(c.x, t, paths, c.seed, antithetic=anti, fresh=fresh, workers=8)
    rep = eng.gradient_of_G(c.x, t, cfg, method="tangent")
    assert_report_close(rep, orc)
    adj = eng.gradient_of_G(c.x, t, cfg)
    assert rep.G == adj.G and rep.means == adj.means and rep.lambda_ == adj.lambda_
    assert rel_err(rep.grad, adj.grad) <= 1e-12


@pytest.mark.parametrize("env", [{"LTG_SAFE": "1"}])
def test_tangent_mode_safe_rerun_bitwise(env):
    import os
    c = configs.cfg3()
    eng = Engine(c.spec)
    cfg = MCConfig(paths=3000, seed=c.seed)
    t = configs.load_targets(c)
    base = eng.gradient_of_G(c.x, t, cfg, method="tangent")
    os.environ.update(env)
    try:
        rep = eng.gradient_of_G(c.x, t, cfg, method="tangent")
    finally:
        for k in env:
            os.environ.pop(k)
    assert rep.to_json() == base.to_json()


def test_tangent_mode_nccl_attached_bitwise():
    from paper_1901_04200_b200.engine import nccl_unique_id
    c = configs.cfg3()
    t = configs.load_targets(c)
    cfg = MCConfig(paths=4099, seed=c.seed)
    base = Engine(c.spec).gradient_of_G(c.x, t, cfg, method="tangent")
    eng = Engine(c.spec)
    eng.attach_nccl(nccl_unique_id(), 0, 1)
    assert eng.gradient_of_G(c.x, t, cfg, method="tangent").to_json() == base.to_json()


def test_tangent_mode_scope(small):
    # grids with several leverage columns (heston_small, cfg2), the basket and
    # fp32 are adjoint-only: refused where the reference would not be matched
    spec, eng = small
    x = eng.pack_params()
    with pytest.raises(ValueError, match="tangent"):
        eng.gradient_of_G(x, [1.0] * eng.m, MCConfig(paths=64, seed=1), method="tangent")
    c = configs.cfg4()
    with pytest.raises(ValueError, match="tangent"):
        Engine(c.spec).gradient_of_G(c.x, c.targets, MCConfig(paths=64, seed=1),
                                     method="tangent")
    c = configs.cfg3()
    with pytest.raises(ValueError, match="tangent"):
        Engine(c.spec).gradient_of_G(c.x, configs.load_targets(c),
                                     MCConfig(paths=64, seed=1, precision=1), method="tangent")


def test_lambda_zero_identity(small):
    # test_calibrate.cpp:201-221: targets = means at the truth, same seed
    spec, eng = small
    x = eng.pack_params()
    cfg = MCConfig(paths=5000, seed=17)
    t = eng.estimate_means(x, cfg).means
    rep = eng.gradient_of_G(x, t, cfg)
    assert rep.G == 0.0
    assert all(v == 0.0 for v in rep.lambda_)
    assert all(v == 0.0 for v in rep.grad)


def test_rerun_bitwise_deterministic(small):
    spec, eng = small
    x = eng.pack_params()
    cfg = MCConfig(paths=70001, seed=3)
    t = [v * 0.9 for v in eng.estimate_means(x, cfg).means]
    a = eng.gradient_of_G(x, t, cfg)
    b = eng.gradient_of_G(x, t, cfg)
    assert a.to_json() == b.to_json()


def test_gpu_fd_matches_adjoint(small):
    # acceptance.cpp:125-154 criterion 1 on the GPU: central differences of G
    # under common random numbers vs the two-pass gradient, 1e-6
    spec, eng = small
    x = eng.pack_params()
    cfg = MCConfig(paths=spec.mc.paths, seed=spec.mc.seed)
    t = [0.9 * v for v in eng.estimate_means(x, cfg).means]
    rep = eng.gradient_of_G(x, t, cfg)
    fd = eng.finite_diff_gradient_of_G(x, t, cfg, 3e-7)
    g = np.asarray(rep.grad)
    assert np.max(np.abs(g - fd) / np.maximum(np.abs(g), 1e-8)) <= 1e-6


def test_report_fields_and_json(small):
    spec, eng = small
    x = eng.pack_params()
    rep = eng.gradient_of_G(x, [1.0] * 4, MCConfig(paths=100, seed=8, memory_mode=MODE_STORE))
    assert rep.paths == 100 and rep.seed == 8 and rep.mode == "store"
    assert list(__import__("json").loads(rep.to_json()).keys()) == \
        ["G", "means", "lambda", "grad", "paths", "mode", "seed"]


def test_error_behaviour(small):
    spec, eng = small
    x = eng.pack_params()
    with pytest.raises(ValueError):
        eng.gradient_of_G(x[:-1], [1.0] * 4, MCConfig(paths=10, seed=1))
    with pytest.raises(ValueError):
        eng.gradient_of_G(x, [1.0] * 3, MCConfig(paths=10, seed=1))
    with pytest.raises(ValueError):
        eng.gradient_of_G(x, [1.0] * 4, MCConfig(paths=0, seed=1))
    with pytest.raises(ValueError):
        eng.gradient_of_G(x, [1.0] * 4, MCConfig(paths=10, seed=1, memory_mode=MODE_STORE,
                                                 fresh_step2_paths=True))
    bad = list(x)
    bad[3] = 1.5  # rho: sqrt(1 - rho^2) of a negative -> EvalError in the reference
    with pytest.raises(EvalError):
        eng.gradient_of_G(bad, [1.0] * 4, MCConfig(paths=10, seed=1))


@pytest.mark.parametrize("j,val", [(0, float("nan")), (4, float("inf")), (2, 1e300)])
def test_nonfinite_values_propagate_like_the_reference(ref, j, val):
    # the reference library's gradient_of_G returns NaN / inf instead of
    # throwing (only a negative sqrt argument is an EvalError); so does the
    # engine: LTG_OK with the same non-finite pattern in means and G, and
    # the finite entries within the usual bar
    c = configs.cfg3()
    prog = ref.program(c.spec)
    t = configs.load_targets(c)
    x = list(c.x)
    x[j] = val
    orc = prog.gradient_of_G(x, t, 2000, c.seed, workers=8)
    rep = Engine(c.spec).gradient_of_G(x, t, MCConfig(paths=2000, seed=c.seed))
    pairs = [(rep.means, orc["means"]), ([rep.G], [orc["G"]])]
    if np.all(np.isfinite(orc["grad"])):
        pairs.append((rep.grad, orc["grad"]))
    for a, b in pairs:
        a, b = np.asarray(a, float), np.asarray(b, float)
        assert np.array_equal(np.isnan(a), np.isnan(b)), (a, b)
        assert np.array_equal(np.isinf(a), np.isinf(b)), (a, b)
        f = np.isfinite(a)
        if f.any():
            assert rel_err(a[f], b[f]) <= TOL


# ------------------------------------- per-chunk parity at full P (§8c) ----

def _chunk_lambda(m):
    return np.array([0.05 * math.sin(1.0 + i) for i in range(m)])


@pytest.mark.parametrize("k,anti", [(0, False), (517, False), (1023, False), (731, True)])
def test_cfg5_chunk_sums_match_reference(ref, k, anti):
    # 2^16-path chunks of config 5 at their place in the full
    # 2^26 path set — the reference's forward_pass / reverse_pass on the same
    # chunk (path_offset = k*2^16) against the GPU's unreduced chunk totals
    c = configs.cfg5()
    eng = Engine(c.spec)
    prog = ref.program(c.spec)
    lam = _chunk_lambda(c.m)
    p0, n = k << 16, 1 << 16
    s1, s2, adj = eng.chunk_sums(c.x, lam, c.seed, anti, p0, n)
    r1, r2 = prog.forward_sums(c.x, c.seed, p0, n, antithetic=anti, workers=os.cpu_count())
    radj = prog.reverse_sums(c.x, c.seed, p0, n, lam, antithetic=anti, workers=os.cpu_count())
    assert rel_err(s1, r1, 1e-12) <= 1e-12
    assert rel_err(s2, r2, 1e-12) <= 1e-12
    assert rel_err(adj, radj) <= TOL, (adj, radj)


def test_cfg4_chunk_sums_match_reference(ref):
    c = configs.cfg4()
    eng = Engine(c.spec)
    prog = ref.program(c.spec)
    lam = _chunk_lambda(c.m)
    p0, n = 3 << 20, 1 << 14
    s1, s2, adj = eng.chunk_sums(c.x, lam, c.seed, False, p0, n)
    r1, r2 = prog.forward_sums(c.x, c.seed, p0, n, workers=os.cpu_count())
    radj = prog.reverse_sums(c.x, c.seed, p0, n, lam, workers=os.cpu_count())
    assert rel_err(s1, r1, 1e-12) <= 1e-12 and rel_err(s2, r2, 1e-12) <= 1e-12
    assert rel_err(adj, radj) <= TOL


def test_cfg5_end_to_end_2p22(ref):
    # config 5's model end to end at P = 2^22 against the
    # reference's gradient_of_G (all host cores; ~30 s of CPU)
    c = configs.cfg5(1 << 22)
    t = configs.load_targets(configs.cfg5())
    prog = ref.program(c.spec)
    orc = prog.gradient_of_G(c.x, t, c.paths, c.seed, workers=os.cpu_count())
    rep = Engine(c.spec).gradient_of_G(c.x, t, MCConfig(paths=c.paths, seed=c.seed))
    assert_report_close(rep, orc)


def test_rare_flag_reruns_exactly(ref):
    # v0 = 1e-300: the first step's sqrt(V) is outside the fast sqrt's exact
    # range (V < 2^-970), which the fast step flags (heston.cu heston_step) —
    # the call must be redone with the exact kernels and still match the
    # reference; a sane call must not rerun
    c = configs.cfg3()
    eng = Engine(c.spec)
    prog = ref.program(c.spec)
    t = configs.load_targets(c)
    cfg = MCConfig(paths=3000, seed=c.seed)
    eng.gradient_of_G(c.x, t, cfg)
    assert eng.timing()["safe_rerun"] == 0
    x = list(c.x)
    x[4] = 1e-300
    orc = prog.gradient_of_G(x, t, 3000, c.seed, workers=8)
    rep = eng.gradient_of_G(x, t, cfg)
    assert eng.timing()["safe_rerun"] == 1
    assert_report_close(rep, orc)
    rep_t = eng.gradient_of_G(x, t, cfg, method="tangent")
    assert eng.timing()["safe_rerun"] == 1
    assert_report_close(rep_t, orc)


@pytest.mark.parametrize("name,paths,seed,anti,fresh,method", [
    ("cfg2", 3001, 42, True, False, "adjoint"),
    ("cfg2", 2048, (1 << 40) + 7, False, True, "adjoint"),
    ("cfg1", 5000, (1 << 63) + 11, True, False, "adjoint"),
    ("cfg1", 4096, (1 << 35) + 3, False, True, "tangent"),
    ("cfg3", 2500, (1 << 50) + 1, True, True, "adjoint"),
    ("cfg3", 2500, (1 << 50) + 1, True, True, "tangent"),
])
def test_option_combinations_match_reference(ref, name, paths, seed, anti, fresh, method):
    # MCConfig options crossed with 64-bit seeds (the Philox key's high word)
    c = configs.ALL[name]()
    eng = Engine(c.spec)
    prog = ref.program(c.spec)
    t = configs.load_targets(c) or _targets_from(prog, c.truth, paths, 4242)
    orc = prog.gradient_of_G(c.x, t, paths, seed, antithetic=anti, fresh=fresh, workers=8)
    rep = eng.gradient_of_G(c.x, t, MCConfig(paths=paths, seed=seed, antithetic=anti,
                                             fresh_step2_paths=fresh), method=method)
    assert_report_close(rep, orc)


def test_single_process_device_group():
    # ltg_create_*_devices: a one-device group (all this environment has) runs
    # every call through the group path (member threads, ncclCommInitAll
    # communicators, the in-place all-gather) and must equal the plain context
    c = configs.cfg3()
    t = configs.load_targets(c)
    cfg = MCConfig(paths=4099, seed=c.seed)
    plain = Engine(c.spec)
    grp = Engine(c.spec, devices=[0])
    assert grp.M == plain.M and grp.m == plain.m and grp.rng_exact
    assert grp.gradient_of_G(c.x, t, cfg).to_json() == plain.gradient_of_G(c.x, t, cfg).to_json()
    assert grp.gradient_of_G(c.x, t, cfg, method="tangent").to_json() == \
        plain.gradient_of_G(c.x, t, cfg, method="tangent").to_json()
    assert grp.estimate_means(c.x, cfg).means == plain.estimate_means(c.x, cfg).means
    assert np.array_equal(grp.fill_normals(7, 8, False, 3, 64), plain.fill_normals(7, 8, False, 3, 64))
    assert grp.timing()["total_ms"] > 0
    from paper_1901_04200_b200.engine import nccl_unique_id
    with pytest.raises(ValueError):
        grp.attach_nccl(nccl_unique_id(), 0, 1)
    b = configs.cfg4()
    bg = Engine(b.spec, devices=[0])
    cfg4 = MCConfig(paths=2048, seed=b.seed)
    assert bg.gradient_of_G(b.x, b.targets, cfg4).to_json() == \
        Engine(b.spec).gradient_of_G(b.x, b.targets, cfg4).to_json()
    with pytest.raises(ValueError):
        Engine(c.spec, devices=[0, 0])


@pytest.mark.parametrize("anti,fresh", [(True, False), (False, True), (True, True)])
def test_fp32_option_combinations(ref, anti, fresh):
    # the fp32 variant under antithetic draws / fresh step-2 paths, at the
    # fp32 tolerances of DESIGN.md §6 against the fp64 reference
    from paper_1901_04200_b200.model import FP32
    c = configs.cfg3()
    t = configs.load_targets(c)
    prog = ref.program(c.spec)
    paths = 1 << 13
    orc = prog.gradient_of_G(c.x, t, paths, c.seed, antithetic=anti, fresh=fresh, workers=8)
    rep = Engine(c.spec).gradient_of_G(c.x, t, MCConfig(paths=paths, seed=c.seed, antithetic=anti,
                                                        fresh_step2_paths=fresh, precision=FP32))
    tol = FP32_TOL["cfg3"]
    assert rel_err(rep.means, orc["means"], 1e-6) <= tol["means"]
    assert rel_err([rep.G], [orc["G"]]) <= tol["G"]
    assert rel_err(rep.grad, orc["grad"], 1e-3) <= tol["grad"]


@pytest.mark.parametrize("world", [2, 3])
def test_multi_rank_paths_on_one_gpu(world):
    # LTG_LOOPBACK=1: `world` member contexts share the GPU and exchange their
    # chunk rows with device copies where NCCL would all-gather, so every
    # rank-dependent piece of the engine (shard plans, per-rank rows and
    # checkpoint tables, the all-gather layout, the rare-flag reduction) runs
    # for real; the reports must equal the one-context engine's bit for bit
    import os
    c = configs.cfg3()
    t = configs.load_targets(c)
    plain = Engine(c.spec)
    os.environ["LTG_LOOPBACK"] = "1"
    try:
        grp = Engine(c.spec, devices=[0] * world)
    finally:
        os.environ.pop("LTG_LOOPBACK")
    for cfg in (MCConfig(paths=50000 + 17, seed=c.seed),
                MCConfig(paths=9001, seed=7, antithetic=True),
                MCConfig(paths=4099, seed=c.seed, fresh_step2_paths=True)):
        assert grp.gradient_of_G(c.x, t, cfg).to_json() == plain.gradient_of_G(c.x, t, cfg).to_json()
        assert grp.gradient_of_G(c.x, t, cfg, method="tangent").to_json() == \
            plain.gradient_of_G(c.x, t, cfg, method="tangent").to_json()
        a, b = grp.estimate_means(c.x, cfg), plain.estimate_means(c.x, cfg)
        assert a.means == b.means and a.std_errors == b.std_errors
    # the rare-flag rerun agreed across ranks
    x = list(c.x)
    x[4] = 1e-300
    cfg = MCConfig(paths=3000, seed=c.seed)
    assert grp.gradient_of_G(x, t, cfg).to_json() == plain.gradient_of_G(x, t, cfg).to_json()
    assert grp.timing()["safe_rerun"] == 1
    # the basket (store-mode pass 2) across ranks
    b4 = configs.cfg4()
    os.environ["LTG_LOOPBACK"] = "1"
    try:
        bg = Engine(b4.spec, devices=[0] * world)
    finally:
        os.environ.pop("LTG_LOOPBACK")
    cfg4 = MCConfig(paths=3001, seed=b4.seed)
    assert bg.gradient_of_G(b4.x, b4.targets, cfg4).to_json() == \
        Engine(b4.spec).gradient_of_G(b4.x, b4.targets, cfg4).to_json()


_UNIT_SCRIPT = r"""
import json, sys
sys.path.insert(0, sys.argv[1])
from paper_1901_04200_b200 import configs
from paper_1901_04200_b200.engine import Engine
from paper_1901_04200_b200.model import MCConfig
c = configs.cfg3()
t = configs.load_targets(c)
eng = Engine(c.spec)
out = {}
for prec in (0, 1):
    for fresh in (False, True):
        cfg = MCConfig(paths=5000, seed=c.seed, precision=prec, fresh_step2_paths=fresh)
        out[f"{prec}{int(fresh)}"] = eng.gradient_of_G(c.x, t, cfg).to_json()
print(json.dumps(out))
"""


def test_unit_leverage_kernels_bitwise_identical():
    # configs 3/5 evaluate at L_0_0 = 1.0: the kLevUnit kernels skip the
    # products by L (exact) — in fp64 the same reports, bit for bit, as the
    # general one-cell kernels (LTG_UNIT_LEV=0), both pass-2 plans. The fp32
    # mode has no bit contract: its forward sums are the same
    # bits too, but the compiler contracts the reverse sweep's float products
    # by L = 1.0f differently in the two instantiations, so its gradient is
    # held to a few float ulps of the general kernel's instead.
    import json
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    runs = []
    for flag in ("1", "0"):
        env = dict(os.environ, LTG_UNIT_LEV=flag)
        r = subprocess.run([sys.executable, "-c", _UNIT_SCRIPT, root], env=env,
                           capture_output=True, text=True, timeout=600)
        assert r.returncode == 0, r.stderr[-2000:]
        runs.append(json.loads(r.stdout.strip().splitlines()[-1]))
    for key in ("00", "01"):
        assert runs[0][key] == runs[1][key], key
    for key in ("10", "11"):
        a, b = json.loads(runs[0][key]), json.loads(runs[1][key])
        assert a["means"] == b["means"] and a["G"] == b["G"], key
        ga, gb = np.asarray(a["grad"]), np.asarray(b["grad"])
        assert np.max(np.abs(ga - gb)) <= 1e-6 * np.max(np.abs(gb)), key


def _short_heston(steps):
    # heston_small's model on a grid of `steps` <= 8 steps: one checkpoint
    # segment, so pass 2 replays nothing before its adjoint sweep
    import copy
    from paper_1901_04200_b200.model import CALL, PUT, Instrument
    spec = copy.deepcopy(load_model_spec(os.path.join(os.path.dirname(__file__), "golden",
                                                      "heston_small.json")))
    spec.mc.steps = steps
    spec.instruments = [Instrument(CALL, 95.0, steps), Instrument(PUT, 100.0, max(1, steps // 2)),
                        Instrument(CALL, 105.0, steps)]
    return spec


@pytest.mark.parametrize("case", ["cfg3", "short"])
def test_fresh_path_set_is_range_checked(ref, monkeypatch, case):
    # With fresh_step2_paths pass 2 runs a path set that pass 1 never saw, so
    # its arguments must be range-checked before the fast adjoint kernel
    # trusts them: the checkpoint replay covers every step (not only up to
    # the last segment), and a one-segment model gets a checking forward.
    # LTG_TEST_FRESH_RARE=1 makes exactly that check flag every path: the
    # call must then rerun with the exact kernels and give the same bits.
    if case == "cfg3":
        c = configs.cfg3()
        spec, x, t, seed = c.spec, c.x, configs.load_targets(c), c.seed
    else:
        spec = _short_heston(6)
        eng0 = Engine(spec)
        x = eng0.pack_params()
        seed = 11
        t = [0.9 * v for v in eng0.estimate_means(x, MCConfig(paths=4000, seed=5)).means]
    eng = Engine(spec)
    paths = 3001
    fresh = MCConfig(paths=paths, seed=seed, fresh_step2_paths=True)
    base = eng.gradient_of_G(x, t, fresh)
    assert eng.timing()["safe_rerun"] == 0
    monkeypatch.setenv("LTG_TEST_FRESH_RARE", "1")
    rep = eng.gradient_of_G(x, t, fresh)
    assert eng.timing()["safe_rerun"] == 1
    assert rep.to_json() == base.to_json()
    # the knob touches only the fresh path set's check
    eng.gradient_of_G(x, t, MCConfig(paths=paths, seed=seed))
    assert eng.timing()["safe_rerun"] == 0
    orc = ref.program(spec).gradient_of_G(x, t, paths, seed, fresh=True, workers=8)
    assert_report_close(rep, orc)
