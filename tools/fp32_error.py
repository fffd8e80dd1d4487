"""Relative error of the fp32 mode against the fp64 reference (development helper)."""
import sys, os, json
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1901_04200_b200 import configs
from paper_1901_04200_b200.engine import Engine
from paper_1901_04200_b200.model import MCConfig, FP32, FP64, load_model_spec
from oracle.bindings import Ref

ref = Ref()
def rel(a, b, floor_frac):
    a, b = np.asarray(a, float), np.asarray(b, float)
    fl = floor_frac * max(np.abs(a).max(), np.abs(b).max())
    return float(np.max(np.abs(a - b) / np.maximum(np.maximum(np.abs(a), np.abs(b)), fl)))
for name, paths in [("cfg3", 1 << 14), ("cfg1", 1 << 16), ("cfg2", 1 << 14)]:
    c = configs.ALL[name]()
    t = configs.load_targets(c)
    prog = ref.program(c.spec)
    orc = prog.gradient_of_G(c.x, t, paths, c.seed, workers=os.cpu_count())
    e = Engine(c.spec)
    r32 = e.gradient_of_G(c.x, t, MCConfig(paths=paths, seed=c.seed, precision=FP32))
    r64 = e.gradient_of_G(c.x, t, MCConfig(paths=paths, seed=c.seed, precision=FP64))
    print(json.dumps({"cfg": name, "paths": paths,
        "fp32_means": rel(r32.means, orc["means"], 1e-6), "fp32_G": rel([r32.G], [orc["G"]], 1e-6),
        "fp32_grad": rel(r32.grad, orc["grad"], 1e-3), "fp32_grad_floor1e-6": rel(r32.grad, orc["grad"], 1e-6),
        "fp64_grad": rel(r64.grad, orc["grad"], 1e-12)}))
    big = 1 << 20
    e.gradient_of_G(c.x, t, MCConfig(paths=big, seed=c.seed, precision=FP32))
    t32 = e.timing()
    e.gradient_of_G(c.x, t, MCConfig(paths=big, seed=c.seed, precision=FP64))
    t64 = e.timing()
    print(name, "2^20 fp32 ms", round(t32["total_ms"], 2), "fp64 ms", round(t64["total_ms"], 2))
