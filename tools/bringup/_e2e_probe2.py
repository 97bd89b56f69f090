# bring-up: device timeline of one end-to-end cd_k_update (host buffers) via events on the RBM stream
import sys, time
sys.path.insert(0, '.')
import numpy as np, torch
from oracle import oracle as O
from paper_1804_04512_b200 import fastnn as F
B, V, H = 100, 784, 500
v0 = torch.empty((B, V), dtype=torch.float32, pin_memory=True).numpy(); v0[:] = O.bernoulli_f32(3, 0.5, B * V).reshape(B, V)
u = torch.empty((B, H), dtype=torch.float64, pin_memory=True).numpy(); u[:] = O.canonical_f64(5, B * H).reshape(B, H)
rbm = F.Rbm(H, V); rbm.init(42)
for _ in range(50): F.cd_k_update(rbm, v0, 1, 0.1, u, B)
s = torch.cuda.ExternalStream(rbm.stream_handle())
lib = F._lib.load()
n = 300
res = []
for mode in ("e2e", "stage_only", "run_only", "run+recon"):
    ts = []
    for i in range(n):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0 = time.perf_counter()
        e0.record(s)
        if mode == "e2e":
            F.cd_k_update(rbm, v0, 1, 0.1, u, B)
        elif mode == "stage_only":
            rbm.stage(v0, u)
        elif mode == "run_only":
            rbm.run_staged(1, 0.1, B)
        else:
            rbm.run_staged(1, 0.1, B); rbm.recon()
        e1.record(s)
        e1.synchronize()
        t1 = time.perf_counter()
        ts.append(((t1 - t0) * 1e6, e0.elapsed_time(e1) * 1e3))
    ts = np.array(ts[20:])
    print(f"{mode:12s} wall {np.median(ts[:,0]):7.1f} us   device(e0->e1) {np.median(ts[:,1]):7.1f} us")
# pure copies
dv = torch.empty((B, V), device='cuda'); du = torch.empty((B, H), dtype=torch.float64, device='cuda')
tv, tu = torch.from_numpy(v0), torch.from_numpy(u)
for name, pairs in (("h2d v0 313KB", [(dv, tv)]), ("h2d u 400KB", [(du, tu)]), ("h2d both", [(dv, tv), (du, tu)])):
    ts = []
    for i in range(200):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        with torch.cuda.stream(s):
            for d, h in pairs: d.copy_(h, non_blocking=True)
        e1.record(s); e1.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3)
    print(f"{name:14s} device {np.median(ts[20:]):6.1f} us")
