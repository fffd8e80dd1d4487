"""CUDA-graph replay of calls (engine.cpp run_body): the second call of a
shape is captured, later ones replay the graph with updated kernel arguments.
Every report must be bit for bit the eager one (LTG_GRAPH=0), across changes
of parameters, targets, seed and path count, for the adjoint, tangent and
means calls, and a shape change must fall back to eager execution."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SCRIPT = r"""
import json, sys
sys.path.insert(0, sys.argv[1])
from paper_1901_04200_b200 import configs
from paper_1901_04200_b200.engine import Engine
from paper_1901_04200_b200.model import MCConfig
out = []
for name, paths in (("cfg1", 1 << 16), ("cfg3", 4099), ("cfg4", 3001)):
    c = configs.ALL[name]()
    t = configs.load_targets(c) or c.targets
    eng = Engine(c.spec)
    x1 = list(c.x)
    # (x2 keeps config 3's unit leverage cell: L = 1.0 selects other kernels)
    x2 = [v * 1.01 for v in c.x[:5]] + list(c.x[5:]) if name == "cfg3" else [v * 1.01 for v in c.x]
    calls = [(x1, 7, paths), (x1, 7, paths), (x1, 7, paths), (x2, 7, paths), (x2, 8, paths),
             (x1, 9, paths + 128), (x1, 9, paths + 128), (x2, 1, paths + 128), (x1, 7, paths)]
    for i, (x, seed, p) in enumerate(calls):
        cfg = MCConfig(paths=p, seed=seed, antithetic=(name == "cfg1"))
        r = eng.gradient_of_G(x, [v * (1 + 0.01 * i) for v in t], cfg)
        tm = eng.timing()
        out.append([name, "grad", r.to_json(), tm["graph"], tm["launches"], tm["total_ms"] > 0])
        if name == "cfg3":
            r = eng.gradient_of_G(x, t, cfg, method="tangent")
            out.append([name, "tangent", r.to_json(), eng.timing()["graph"], 0, True])
        m = eng.estimate_means(x, cfg)
        out.append([name, "means", json.dumps([m.means, m.std_errors]), eng.timing()["graph"], 0,
                    True])
print(json.dumps(out))
"""


def _run(flag):
    env = dict(os.environ, LTG_GRAPH=flag)
    r = subprocess.run([sys.executable, "-c", SCRIPT, ROOT], env=env, capture_output=True,
                       text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]
    return json.loads(r.stdout.strip().splitlines()[-1])


def test_graph_replay_is_bitwise_eager():
    eager, graph = _run("0"), _run("1")
    assert len(eager) == len(graph)
    for e, g in zip(eager, graph):
        assert e[:3] == g[:3], (e[:2], e[2][:200], g[2][:200])
        assert e[3] == 0 and e[5] and g[5]
    modes = [g[3] for g in graph if g[1] == "grad"]
    # per config: eager, capture, replay, replay (new x), replay (new seed),
    # eager (new path count), capture, replay, replay (the first shape's
    # graph, kept beside the second's and the means calls')
    for k in range(3):
        assert modes[9 * k:9 * k + 9] == [0, 1, 2, 2, 2, 0, 1, 2, 2], modes
    # the same kernels run either way
    assert [g[4] for g in graph] == [e[4] for e in eager]
