"""Generate tests/golden/*.json from the REFERENCE library compiled in place
(oracle/_ref/libltref.so). The fixtures pin the plain-C restatement
(oracle/lt_oracle.c) bit for bit on machines where /root/reference is absent.
Doubles are stored as float.hex() strings so they survive JSON exactly."""
import json, os, sys
import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1901_04200_b200 import configs
from paper_1901_04200_b200.model import load_model_spec
from oracle.bindings import Ref

G = os.path.join(ROOT, "tests", "golden")
ref = Ref()


def hx(a):
    return [float(v).hex() for v in np.ravel(a)]


rng = {"philox": [], "uniform": [], "as241": [], "draws": []}
for ctr, key in [([0, 0, 0, 0], [0, 0]),
                 ([0xffffffff] * 4, [0xffffffff] * 2),
                 ([0x243f6a88, 0x85a308d3, 0x13198a2e, 0x03707344], [0xa4093822, 0x299f31d0])]:
    rng["philox"].append({"ctr": ctr, "key": key, "out": ref.philox_block(ctr, key)})
for w0, w1 in [(0, 0), (0xffffffff, 0xffffffff), (0x12345678, 0x9abcdef0)]:
    rng["uniform"].append({"w": [w0, w1], "u": ref.uniform(w0, w1).hex()})
for p in [0.5, 0.025, 0.975, 1e-10, 0.9999999999, 0.31830988618, 0.841344746068543, 0.07,
          0.93, 2.0 ** -53, 1 - 2.0 ** -53, 1e-300]:
    rng["as241"].append({"p": p.hex(), "z": ref.inverse_normal_cdf(p).hex()})
for seed, dim, anti, path0, n in [(42, 8, False, 7, 1), (20190114, 1512, False, 0, 4),
                                  (77, 4, True, 0, 6), (31415, 33, True, (1 << 40) + 3, 5),
                                  ((1 << 63) + 12345, 128, False, (1 << 33) + 17, 8),
                                  (2718, 64, False, 1 << 20, 32)]:
    z = ref.fill_normals(seed, dim, anti, path0, n)
    rng["draws"].append({"seed": seed, "dim": dim, "antithetic": anti, "path0": path0,
                         "npaths": n, "z": hx(z)})
with open(os.path.join(G, "rng_golden.json"), "w") as f:
    json.dump(rng, f)

cases = []
small = load_model_spec(os.path.join(G, "heston_small.json"))
specs = [("heston_small", small, None, None, 64), ("heston_small", small, None, None, 1001)]
for name, P in [("cfg1", 4096), ("cfg2", 1024), ("cfg3", 256), ("cfg4", 256)]:
    c = configs.ALL[name]()
    specs.append((name, c.spec, c.x, c.targets, P))
for name, spec, x, targets, P in specs:
    prog = ref.program(spec)
    if x is None:
        x = prog.initial_params()
    if targets is None:
        targets = 0.9 * prog.estimate_means(x, P, 4242, lane_width=8)[0]
    r = prog.gradient_of_G(x, targets, P, 42, lane_width=8, workers=1)
    means, se = prog.estimate_means(x, P, 42, lane_width=8)
    cases.append({"name": name, "paths": P, "seed": 42, "lane_width": 8, "x": hx(x),
                  "targets": hx(targets), "G": float(r["G"]).hex(), "means": hx(r["means"]),
                  "lambda": hx(r["lambda_"]), "grad": hx(r["grad"]), "std_errors": hx(se)})
with open(os.path.join(G, "ref_gradients.json"), "w") as f:
    json.dump({"generator": "oracle/_ref gradient_of_G (reference headers, -O3 -fno-math-errno)",
               "cases": cases}, f)
print("ok", len(cases))
