"""Host-side overhead of one gradient_of_G call (development helper)."""
import sys, time
sys.path.insert(0, '.')
from paper_1901_04200_b200 import configs
from paper_1901_04200_b200.engine import Engine
from paper_1901_04200_b200.model import MCConfig
import ctypes as C, numpy as np
c = configs.cfg1()
eng = Engine(c.spec)
t = configs.load_targets(c) or [1.0] * c.m
cfg = MCConfig(paths=c.paths, seed=c.seed)
for _ in range(5): eng.gradient_of_G(c.x, t, cfg)
N = 200
t0 = time.perf_counter()
for _ in range(N): eng.gradient_of_G(c.x, t, cfg)
w = (time.perf_counter() - t0) / N
tm = eng.timing()
print("cfg1 grad: wall/call %.3f ms, device total %.3f ms, launches %d" % (w * 1e3, tm["total_ms"], tm["launches"]))
t0 = time.perf_counter()
for _ in range(N): eng.estimate_means(c.x, cfg)
print("cfg1 means: wall/call %.3f ms" % ((time.perf_counter() - t0) / N * 1e3))
cfg2 = MCConfig(paths=128, seed=c.seed)
for _ in range(3): eng.gradient_of_G(c.x, t, cfg2)
t0 = time.perf_counter()
for _ in range(N): eng.gradient_of_G(c.x, t, cfg2)
w = (time.perf_counter() - t0) / N
tm = eng.timing()
print("128 paths grad: wall/call %.3f ms, device total %.3f ms" % (w * 1e3, tm["total_ms"]))
# raw ctypes call overhead
from paper_1901_04200_b200 import cabi
x = np.ascontiguousarray(c.x, dtype=np.float64); tt = np.ascontiguousarray(t, dtype=np.float64)
means, lam, grad = np.empty(c.m), np.empty(c.m), np.empty(len(c.x))
dp = C.POINTER(C.c_double)
rep = cabi.ReportC(0.0, means.ctypes.data_as(dp), lam.ctypes.data_as(dp), grad.ctypes.data_as(dp), None, 0, 0, 0)
cc = cabi.MCConfigC(128, c.seed, 0, 0, 0, 0)
L = eng.lib
t0 = time.perf_counter()
for _ in range(N): L.ltg_gradient_of_G(eng.h, x.ctypes.data_as(dp), x.size, tt.ctypes.data_as(dp), tt.size, C.byref(cc), C.byref(rep))
print("128 paths raw C call: %.3f ms" % ((time.perf_counter() - t0) / N * 1e3))
