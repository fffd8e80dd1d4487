"""Wall vs device time per gradient_of_G call on cfg3 (development helper)."""
import sys, time
sys.path.insert(0, '.')
from paper_1901_04200_b200 import configs
from paper_1901_04200_b200.engine import Engine
from paper_1901_04200_b200.model import MCConfig
c = configs.cfg3()
eng = Engine(c.spec)
t = configs.load_targets(c)
for paths in (1 << 20, 1 << 16):
    cfg = MCConfig(paths=paths, seed=c.seed)
    for _ in range(3): eng.gradient_of_G(c.x, t, cfg)
    N = 20
    dev = 0.0
    t0 = time.perf_counter()
    for _ in range(N):
        eng.gradient_of_G(c.x, t, cfg)
        dev += eng.timing()["total_ms"]
    w = (time.perf_counter() - t0) / N * 1e3
    print(f"paths {paths}: wall {w:.3f} ms/call, device {dev / N:.3f} ms/call, host {w - dev / N:.3f}")
