"""Pipeline fill of the streamed RBM loop: device time of one train_stream call vs its step count
(device-resident batches + uniforms, and host batches + device draws), plus the host time of the call."""
import sys
import time
import numpy as np
import torch
sys.path.insert(0, ".")
from paper_1804_04512_b200 import fastnn as F

B, H, V = 100, 500, 784
r = F.Rbm(H, V)
r.init(1)
N = 200
dev = torch.device("cuda", 0)
v = (torch.rand(N * B, V, device=dev) < 0.5).float()
u = torch.rand(N * B, H, device=dev, dtype=torch.float64)
vh = torch.empty(N * B, V, dtype=torch.float32).pin_memory()
vh.copy_(v.cpu())
s = torch.cuda.ExternalStream(r.stream_handle())
g = F.Mt19937(3)


def run(fn):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record(s)
    t0 = time.perf_counter()
    fn()
    t1 = time.perf_counter()
    e1.record(s)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) * 1e3, (t1 - t0) * 1e6


for K in (1, 2, 5, 10, 20, 50, 200):
    for _ in range(2):
        r.train_stream_ptr(v.data_ptr(), u.data_ptr(), K, B, 0.1)
        r.train_stream(vh.numpy()[:K * B], g, B, 0.1)
    a = min(run(lambda: r.train_stream_ptr(v.data_ptr(), u.data_ptr(), K, B, 0.1)) for _ in range(3))
    b = min(run(lambda: r.train_stream(vh.numpy()[:K * B], g, B, 0.1)) for _ in range(3))
    print(f"K={K:4d}  value: {a[0]:8.1f} us ({a[0] / K:6.1f}/step, host {a[1]:8.1f})   "
          f"e2e: {b[0]:8.1f} us ({b[0] / K:6.1f}/step, host {b[1]:8.1f})")

# decomposition at K = 1 and 20: host batches + host uniforms; device batches + device draws
uh = torch.empty(N * B, H, dtype=torch.float64).pin_memory()
uh.copy_(u.cpu())
for K in (1, 20):
    def dev_draws():
        r.set_rng(g)
        r.train_stream_ptr(v.data_ptr(), 0, K, B, 0.1)
        r.get_rng(g)
    for _ in range(2):
        r.train_stream(vh.numpy()[:K * B], uh.numpy()[:K * B], B, 0.1)
        dev_draws()
    a = min(run(lambda: r.train_stream(vh.numpy()[:K * B], uh.numpy()[:K * B], B, 0.1)) for _ in range(3))
    b = min(run(dev_draws) for _ in range(3))
    c = min(run(lambda: (r.set_rng(g), r.get_rng(g))) for _ in range(3))
    print(f"K={K}: host v + host u {a[0]:.1f} us;  device v + device draws {b[0]:.1f} us;  set+get rng {c[0]:.1f} us")
