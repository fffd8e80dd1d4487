"""Small single-GPU calls (engine.cpp "lean calls", finish.cuh fused_tail):
the pass launches reduce their own chunk tables when these are small (the
last CTA runs launch_reduce_chunks' fixed-order sums), x / targets travel as
kernel arguments, and the call's last kernel publishes the report into the
caller's pinned buffer and clears the rare flag. Every report must equal, bit
for bit, the separate-reduction form (LTG_FUSE_REDUCE=0), and the rare flag a
call leaves behind must never leak into the next call."""
import json
import os
import subprocess
import sys

import numpy as np
import pytest

from paper_1901_04200_b200 import configs
from paper_1901_04200_b200.engine import Engine
from paper_1901_04200_b200.model import MCConfig

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SCRIPT = r"""
import json, os, sys
sys.path.insert(0, sys.argv[1])
from paper_1901_04200_b200 import configs
from paper_1901_04200_b200.engine import Engine
from paper_1901_04200_b200.model import MCConfig, load_model_spec
out = []
small = load_model_spec(os.path.join(sys.argv[1], "tests", "golden", "heston_small.json"))
cases = [("cfg1", configs.cfg1().spec, configs.cfg1().x, None, 1 << 16),
         ("cfg1", configs.cfg1().spec, configs.cfg1().x, None, 1000),
         ("cfg2", configs.cfg2().spec, configs.cfg2().x, None, 4096),
         ("cfg4", configs.cfg4().spec, configs.cfg4().x, configs.cfg4().targets, 3001),
         ("small", small, None, None, 2053)]
for name, spec, x, t, paths in cases:
    eng = Engine(spec)
    x = list(x) if x is not None else list(eng.pack_params())
    if t is None:
        t = [0.9 * v for v in eng.estimate_means(x, MCConfig(paths=4096, seed=5)).means]
    for anti in (False, True):
        for i in range(3):  # eager, capture, replay
            cfg = MCConfig(paths=paths, seed=11 + i, antithetic=anti)
            r = eng.gradient_of_G(x, t, cfg)
            out.append([name, "grad", r.to_json(), eng.timing()["launches"]])
            m = eng.estimate_means(x, cfg)
            out.append([name, "means", json.dumps([m.means, m.std_errors]),
                        eng.timing()["launches"]])
        if name == "cfg1":
            r = eng.gradient_of_G(x, t, cfg, method="tangent")
            out.append([name, "tangent", r.to_json(), eng.timing()["launches"]])
print(json.dumps(out))
"""


def _run(flag):
    env = dict(os.environ, LTG_FUSE_REDUCE=flag)
    r = subprocess.run([sys.executable, "-c", SCRIPT, ROOT], env=env, capture_output=True,
                       text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]
    return json.loads(r.stdout.strip().splitlines()[-1])


def test_fused_reduction_is_bitwise_the_separate_one():
    sep, fused = _run("0"), _run("1")
    assert len(sep) == len(fused)
    for s, f in zip(sep, fused):
        assert s[:3] == f[:3], (s[:2], s[2][:200], f[2][:200])
    # the small tables did fuse: two launches per gradient call (pass 1, pass
    # 2) and one per means call, against 2 + 2 reductions each otherwise
    grads = [(s[3], f[3]) for s, f in zip(sep, fused) if f[0] == "cfg1" and f[1] == "grad"]
    assert all(f == 2 and s == 6 for s, f in grads), grads
    means = [(s[3], f[3]) for s, f in zip(sep, fused) if f[0] == "cfg1" and f[1] == "means"]
    assert all(f == 1 and s == 3 for s, f in means), means


def test_rare_flag_does_not_leak_into_the_next_call():
    # a call whose paths raise the rare flag reruns exactly; the flag it
    # leaves (cleared by the lean call's last kernel, or left set by a
    # non-lean entry point) must not make the next call rerun
    c = configs.cfg1()
    eng, ref = Engine(c.spec), Engine(c.spec)
    t = configs.load_targets(c) or c.targets
    cfg = MCConfig(paths=5000, seed=3)
    x_rare = list(c.x)
    x_rare[4] = 1e-300  # V0 below the fast sqrt's range: every path flags
    expect = ref.gradient_of_G(c.x, t, cfg).to_json()
    for step in range(3):
        r = eng.gradient_of_G(x_rare, t, cfg)
        assert eng.timing()["safe_rerun"] == 1
        assert r.to_json() == ref.gradient_of_G(x_rare, t, cfg).to_json()
        r = eng.gradient_of_G(c.x, t, cfg)
        assert eng.timing()["safe_rerun"] == 0, step
        assert r.to_json() == expect
        # a non-lean entry point whose kernels set the flag, then lean calls
        p = eng.path_payoffs(x_rare, 3, False, 0, 256)
        assert np.isfinite(p).all()
        m = eng.estimate_means(c.x, cfg)
        assert eng.timing()["safe_rerun"] == 0
        assert m.means == ref.estimate_means(c.x, cfg).means


@pytest.mark.parametrize("m,rows,cols,paths", [(64, 4, 8, 3000), (65, 4, 8, 3000),
                                               (80, 6, 6, 2500), (80, 6, 6, 1 << 17)])
def test_models_beyond_the_by_value_arguments(ref, golden_dir, m, rows, cols, paths):
    # up to 32 leverage cells and 64 targets travel in the launch arguments;
    # larger models take the one-copy route through d_x — both against the
    # reference, with the fused (small) and the separate (2^17) reduction
    import copy
    from paper_1901_04200_b200.model import CALL, PUT, Instrument, load_model_spec
    from test_gpu_parity import assert_report_close
    spec = copy.deepcopy(load_model_spec(os.path.join(golden_dir, "heston_small.json")))
    g = np.random.default_rng(m * 1000 + rows)
    steps = spec.mc.steps
    spec.grid.t_nodes = [i * steps * spec.mc.dt / rows for i in range(rows)]
    spec.grid.s_nodes = [float(v) for v in np.linspace(70.0, 130.0, cols)]
    spec.grid.values = [float(v) for v in g.uniform(0.6, 1.4, rows * cols)]
    spec.instruments = [Instrument(int(g.choice([CALL, PUT])), float(g.uniform(80.0, 120.0)),
                                   int(g.integers(1, steps + 1))) for _ in range(m)]
    eng = Engine(spec)
    prog = ref.program(spec)
    x = prog.initial_params()
    assert len(x) == 5 + rows * cols
    means, _ = prog.estimate_means(x, 4096, 77, workers=8)
    targets = 0.95 * means
    orc = prog.gradient_of_G(x, targets, paths, 11, workers=8)
    for _ in range(3):  # eager, capture, replay
        rep = eng.gradient_of_G(x, targets, MCConfig(paths=paths, seed=11))
        assert_report_close(rep, orc)
