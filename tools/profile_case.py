"""One warm gradient_of_G call on a BASELINE config (target of ncu captures)."""
import argparse, json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1901_04200_b200 import configs
from paper_1901_04200_b200.engine import Engine
from paper_1901_04200_b200.model import MCConfig, FP32, FP64

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="cfg3")
ap.add_argument("--paths", type=int, default=1 << 18)
ap.add_argument("--reps", type=int, default=1)
ap.add_argument("--precision", default="fp64")
a = ap.parse_args()
c = configs.ALL[a.config]()
eng = Engine(c.spec)
t = configs.load_targets(c) or [1.0] * c.m
mc = MCConfig(paths=a.paths, seed=c.seed, precision=FP32 if a.precision == "fp32" else FP64)
for _ in range(a.reps):
    rep = eng.gradient_of_G(c.x, t, mc)
print(json.dumps({"config": a.config, "paths": a.paths, "G": rep.G, **eng.timing()}))
