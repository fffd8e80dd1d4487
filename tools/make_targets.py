"""Compute the committed calibration targets of BASELINE configs 2 and 3
(separate-seed forward runs at the truth, 2^22 paths) with the REFERENCE
library itself (oracle/_ref), i.e. synthetic_targets (calibrate.hpp:224-227)
= estimate_means(tape, truth, MCConfig{paths=2^22, seed=TARGET_SEED}).
Run here (needs /root/reference or a built oracle/_ref)."""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1901_04200_b200 import configs
from oracle.bindings import Ref

ref = Ref()
for name in sys.argv[1:] or ["cfg2", "cfg3"]:
    c = configs.ALL[name]()
    prog = ref.program(c.spec)
    t0 = time.time()
    means, se = prog.estimate_means(c.truth, configs.TARGET_PATHS, configs.TARGET_SEED,
                                    lane_width=8, workers=os.cpu_count())
    out = {"config": c.name, "truth": c.truth, "paths": configs.TARGET_PATHS,
           "seed": configs.TARGET_SEED, "generator": "reference estimate_means (oracle/_ref)",
           "targets": [float(v) for v in means], "std_errors": [float(v) for v in se]}
    with open(configs.targets_path(c.name), "w") as f:
        json.dump(out, f, indent=1)
    print(name, f"{time.time() - t0:.1f}s")
