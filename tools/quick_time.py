"""Ad-hoc timing of the engine on BASELINE configs (development helper)."""
import sys, time, json
import numpy as np
sys.path.insert(0, '.')
from paper_1901_04200_b200 import configs
from paper_1901_04200_b200.engine import Engine
from paper_1901_04200_b200.model import MCConfig

names = sys.argv[1:] or ["cfg1", "cfg2", "cfg3"]
for name in names:
    # "cfg3:fp32" -> the fp32 mode
    name, _, prec = name.partition(":")
    c = configs.ALL[name]()
    eng = Engine(c.spec)
    t = configs.load_targets(c) or [1.0] * c.m
    cfg = MCConfig(paths=c.paths, seed=c.seed, precision=1 if prec == "fp32" else 0)
    eng.gradient_of_G(c.x, t, cfg)
    best = None
    for _ in range(3):
        t0 = time.perf_counter(); rep = eng.gradient_of_G(c.x, t, cfg); dt = time.perf_counter() - t0
        tm = eng.timing()
        best = tm if best is None or tm["total_ms"] < best["total_ms"] else best
    print(json.dumps({"cfg": name + (":" + prec if prec else ""), "paths": c.paths, "wall_s": dt, "paths_per_s": c.paths / (best["total_ms"] / 1e3), **best, "G": rep.G}))
