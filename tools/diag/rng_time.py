"""Device generator timing: one Rbm.stage(v0, None) = the mt19937 words kernel + the canonical
kernel for B*H draws (run under ncu for per-kernel durations)."""
import sys
import numpy as np
sys.path.insert(0, ".")
from paper_1804_04512_b200 import fastnn as F

B, H, V = 100, 500, 784
r = F.Rbm(H, V)
r.init(1)
g = F.Mt19937(5)
r.set_rng(g)
v0 = np.zeros((B, V), np.float32)
for _ in range(5):
    r.stage(v0, None)
r.get_rng(g)
m = F.Crbm(1, 28, 28, 12, 5, 5)
m.init(1)
m.set_rng(g)
for _ in range(3):
    m.stage(np.zeros((B, 1, 28, 28), np.float32), None)
m.get_rng(g)
print("ok")
