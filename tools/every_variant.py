"""Small calls that launch every kernel variant of the engine at least once
(development check; `python tools/every_variant.py` exits non-zero on any
engine error). Written for compute-sanitizer, which this GPU pool does not
allow; the variants' results are covered by the parity suites.

Heston pass 1 / pass 2 for the three leverage layouts (one cell, time rows,
rows x columns), fast and SAFE arithmetic, checkpoint intervals 8 and 16, the
draw store, the no-table wave replay (fresh step-2 paths), fp32, the tangent
kernel, caller draws, the basket (store and recompute), the reductions, the
normal generator and the AS241 entry point.
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1901_04200_b200 import configs  # noqa: E402
from paper_1901_04200_b200.engine import Engine  # noqa: E402
from paper_1901_04200_b200.model import (FP32, BufferDrawSource, MCConfig,  # noqa: E402
                                         load_model_spec)

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def shrink(spec, steps):
    spec.mc.steps = steps
    for i in spec.instruments:
        i.maturity_step = min(i.maturity_step, steps)
    return spec


def heston_cases():
    small = load_model_spec(os.path.join(ROOT, "tests", "golden", "heston_small.json"))
    yield "heston_small (grid)", small
    c1 = configs.cfg1()
    yield "cfg1 (time rows)", c1.spec
    c3 = configs.cfg3()
    yield "cfg3 (one cell, 40 steps)", shrink(c3.spec, 40)


def main():
    paths = 1000
    for name, spec in heston_cases():
        eng = Engine(spec)
        x = eng.pack_params()
        t = np.full(eng.m, 1.0)
        for ks in ("8", "16"):
            os.environ["LTG_CKPT_STEPS"] = ks
            for safe in ("0", "1"):
                os.environ["LTG_SAFE"] = safe
                eng.gradient_of_G(x, t, MCConfig(paths=paths, seed=3))
                eng.gradient_of_G(x, t, MCConfig(paths=paths, seed=3, antithetic=True))
            os.environ.pop("LTG_SAFE")
        os.environ.pop("LTG_CKPT_STEPS")
        os.environ["LTG_ZSTORE"] = "0"
        eng.gradient_of_G(x, t, MCConfig(paths=paths + 7, seed=4))
        os.environ.pop("LTG_ZSTORE")
        eng.gradient_of_G(x, t, MCConfig(paths=paths, seed=5, fresh_step2_paths=True))
        try:  # (fp32 gradients need the Feller condition)
            eng.gradient_of_G(x, t, MCConfig(paths=paths, seed=5, precision=FP32))
        except ValueError:
            pass
        eng.estimate_means(x, MCConfig(paths=paths, seed=6))
        try:
            eng.gradient_of_G(x, t, MCConfig(paths=paths, seed=7), method="tangent")
        except ValueError:
            pass  # grid models: adjoint only
        z = np.random.default_rng(1).standard_normal((2 * paths, eng.N))
        eng.gradient_of_G(x, t, MCConfig(paths=paths, fresh_step2_paths=True),
                          source=BufferDrawSource(z, eng.N))
        eng.chunk_sums(x, t, 8, False, 12345, 300)
        eng.path_payoffs(x, 9, False, 0, 64)
        eng.fill_normals(10, 33, True, 5, 100)
        print("ok", name, flush=True)
    eng.inverse_normal(np.array([2.0 ** -53, 1e-12, 0.02, 0.5 + 2.0 ** -53, 0.97, 1 - 2.0 ** -53]))
    b = configs.cfg4(paths)
    be = Engine(b.spec)
    for fresh in (False, True):
        be.gradient_of_G(b.x, b.targets, MCConfig(paths=paths, seed=11, fresh_step2_paths=fresh))
    zb = np.random.default_rng(2).standard_normal((paths, be.N))
    be.gradient_of_G(b.x, b.targets, MCConfig(paths=paths), source=BufferDrawSource(zb, be.N))
    print("ok basket", flush=True)


if __name__ == "__main__":
    main()
