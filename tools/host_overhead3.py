"""Where the time of a small gradient_of_G call goes (cfg1, 2^16 paths):
Python API wall, raw ctypes wall, device event span and its parts
(development helper)."""
import ctypes as C
import sys
import time

import numpy as np

sys.path.insert(0, '.')
from paper_1901_04200_b200 import configs  # noqa: E402
from paper_1901_04200_b200.cabi import ReportC  # noqa: E402
from paper_1901_04200_b200.engine import Engine, _cfg, _p  # noqa: E402
from paper_1901_04200_b200.model import MCConfig  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "cfg1"
c = configs.ALL[name]()
eng = Engine(c.spec)
t = np.asarray(configs.load_targets(c) or c.targets, dtype=float)
x = np.asarray(c.x, dtype=float)
cfg = MCConfig(paths=c.spec.mc.paths if hasattr(c.spec, "mc") else 1 << 16, seed=c.seed)
for _ in range(5):
    eng.gradient_of_G(x, t, cfg)
N = 200
t0 = time.perf_counter()
dev = p1 = p2 = red = 0.0
for _ in range(N):
    eng.gradient_of_G(x, t, cfg)
    tm = eng.timing()
    dev += tm["total_ms"]; p1 += tm["pass1_ms"]; p2 += tm["pass2_ms"]; red += tm["reduce_ms"]
w_api = (time.perf_counter() - t0) / N * 1e3
means, lam, grad = np.empty(eng.m), np.empty(eng.m), np.empty(eng.M)
rep = ReportC(0.0, _p(means), _p(lam), _p(grad), None, 0, 0, 0)
cc = _cfg(cfg)
fn = eng.lib.ltg_gradient_of_G
args = (eng.h, _p(x), x.size, _p(t), t.size, C.byref(cc), C.byref(rep))
t0 = time.perf_counter()
for _ in range(N):
    fn(*args)
w_raw = (time.perf_counter() - t0) / N * 1e3
print(f"{name} paths {cfg.paths}: api wall {w_api:.4f} ms, raw ctypes wall {w_raw:.4f} ms, "
      f"device {dev / N:.4f} ms (pass1 {p1 / N:.4f}, pass2 {p2 / N:.4f}, reduce {red / N:.4f}), "
      f"launches {eng.timing()['launches']}")
