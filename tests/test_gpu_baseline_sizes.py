"""GPU parity at the BASELINE sizes: every config's full path count against the
reference library compiled in place (oracle/_ref), end to end through the C ABI.

  config 1   GBM, 2^16 paths                (test_gpu_parity.py: test_baseline_configs_gradient)
  config 2   local-vol 8x5 grid, 2^20 paths  (here)
  config 3   Heston, 2^20 paths              (here)
  config 4   16-asset basket, 2^22 paths     (here)
  config 5   Heston, 2^26 paths: 16 seeded 2^16-path chunks at their place in the
             full path set, plain and antithetic (here), plus 2^22 end to end
             (test_gpu_parity.py: test_cfg5_end_to_end_2p22)

The reference's gradient_of_G runs with every host core (MCConfig{lane_width=8,
worker_threads=os.cpu_count()}, expectation.hpp:300-344); its result does not
depend on the worker count (BatchSums, expectation.hpp:105-122). The bar is the
north_star's: relative error <= 1e-10 in E[y], lambda, G and grad, with the
denominator max(|a|, |b|, 1e-12 * max|vector|). The residual differences are
summation order only (the GPU's per-path payoffs and adjoints are the
reference's bit for bit), which is why the largest path counts are where the
bar has to be shown.
"""
import os

import numpy as np
import pytest

from paper_1901_04200_b200 import configs
from paper_1901_04200_b200.engine import Engine
from paper_1901_04200_b200.model import MCConfig

pytestmark = pytest.mark.gpu

TOL = 1e-10
WORKERS = os.cpu_count() or 1


def rel_err(a, b, floor_frac=1e-12):
    a, b = np.asarray(a, dtype=float), np.asarray(b, dtype=float)
    floor = floor_frac * max(np.max(np.abs(a)), np.max(np.abs(b)), 1e-300)
    return float(np.max(np.abs(a - b) / np.maximum(np.maximum(np.abs(a), np.abs(b)), floor)))


def _check(rep, orc):
    errs = {"means": rel_err(rep.means, orc["means"]), "lambda": rel_err(rep.lambda_, orc["lambda_"]),
            "G": rel_err([rep.G], [orc["G"]]), "grad": rel_err(rep.grad, orc["grad"])}
    assert max(errs.values()) <= TOL, errs


@pytest.mark.parametrize("name,paths", [("cfg2", 1 << 20), ("cfg3", 1 << 20), ("cfg4", 1 << 22)])
def test_baseline_size_gradient_matches_reference(ref, name, paths):
    c = configs.ALL[name]()
    assert c.paths == paths  # the BASELINE path count of the config
    t = configs.load_targets(c)
    if t is None:
        t = c.targets
    prog = ref.program(c.spec)
    orc = prog.gradient_of_G(c.x, t, paths, c.seed, workers=WORKERS)
    rep = Engine(c.spec).gradient_of_G(c.x, t, MCConfig(paths=paths, seed=c.seed))
    _check(rep, orc)


@pytest.mark.parametrize("name,paths", [("cfg2", 1 << 20), ("cfg3", 1 << 20)])
def test_baseline_size_estimate_means_matches_reference(ref, name, paths):
    c = configs.ALL[name]()
    prog = ref.program(c.spec)
    means, se = prog.estimate_means(c.x, paths, c.seed, workers=WORKERS)
    r = Engine(c.spec).estimate_means(c.x, MCConfig(paths=paths, seed=c.seed))
    assert rel_err(r.means, means) <= TOL
    # standard errors: sqrt(max(0, (sumsq - P*mean^2)/(P-1)))/P, cancellation-limited
    assert rel_err(r.std_errors, se, 1e-9) <= 1e-8


def _cfg5_chunks():
    # 16 seeded chunk indices of config 5's 1024 chunks of 2^16 paths (seed
    # 5005), the first 12 plain and the last 4 antithetic, plus both ends
    rng = np.random.default_rng(5005)
    ks = sorted(int(k) for k in rng.choice(np.arange(1, 1023), size=14, replace=False))
    cases = [(0, False), (1023, False)] + [(k, False) for k in ks[:10]]
    cases += [(k, True) for k in ks[10:]]
    return cases


@pytest.mark.parametrize("k,anti", _cfg5_chunks())
def test_cfg5_seeded_chunks_match_reference(ref, k, anti):
    # per-chunk parity at full P. The GPU's unreduced chunk
    # totals (ltg_chunk_sums) against the reference's forward_pass /
    # reverse_pass on the same global paths (path_offset = k * 2^16,
    # expectation.hpp:152-154, 204-208), seeded with a fixed lambda
    c = configs.cfg5()
    eng = Engine(c.spec)
    prog = ref.program(c.spec)
    lam = np.array([0.05 * np.sin(1.0 + i) for i in range(c.m)])
    p0, n = k << 16, 1 << 16
    s1, s2, adj = eng.chunk_sums(c.x, lam, c.seed, anti, p0, n)
    r1, r2 = prog.forward_sums(c.x, c.seed, p0, n, antithetic=anti, workers=WORKERS)
    radj = prog.reverse_sums(c.x, c.seed, p0, n, lam, antithetic=anti, workers=WORKERS)
    assert rel_err(s1, r1) <= 1e-12
    assert rel_err(s2, r2) <= 1e-12
    assert rel_err(adj, radj) <= TOL, (adj, radj)
