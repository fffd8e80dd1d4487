"""One tangent-mode gradient_of_G call on cfg3 (target of ncu captures)."""
import sys, json
sys.path.insert(0, '.')
from paper_1901_04200_b200 import configs
from paper_1901_04200_b200.engine import Engine
from paper_1901_04200_b200.model import MCConfig
c = configs.cfg3()
eng = Engine(c.spec)
t = configs.load_targets(c)
import os
rep = eng.gradient_of_G(c.x, t, MCConfig(paths=int(os.environ.get("LTG_PATHS", 1 << 18)), seed=c.seed), method="tangent")
print(json.dumps(eng.timing()))
