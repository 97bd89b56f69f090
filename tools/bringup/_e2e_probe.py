# bring-up: where the end-to-end (host buffers) RBM step time goes
import sys, time
sys.path.insert(0, '.')
import numpy as np, torch
from oracle import oracle as O
from paper_1804_04512_b200 import fastnn as F
B, V, H = 100, 784, 500
v0 = torch.empty((B, V), dtype=torch.float32, pin_memory=True).numpy(); v0[:] = O.bernoulli_f32(3, 0.5, B * V).reshape(B, V)
u = torch.empty((B, H), dtype=torch.float64, pin_memory=True).numpy(); u[:] = O.canonical_f64(5, B * H).reshape(B, H)
rbm = F.Rbm(H, V); rbm.init(42)
for _ in range(20): F.cd_k_update(rbm, v0, 1, 0.1, u, B)
torch.cuda.synchronize()
n = 200
t = time.perf_counter()
for _ in range(n): F.cd_k_update(rbm, v0, 1, 0.1, u, B)
print("api call wall us/step %.1f" % ((time.perf_counter() - t) / n * 1e6))
rbm.stage(v0, u)
t = time.perf_counter()
for _ in range(n): rbm.run_staged(1, 0.1, B)
torch.cuda.synchronize()
print("device-resident run_staged wall us/step %.1f" % ((time.perf_counter() - t) / n * 1e6))
dv = torch.empty((B, V), device='cuda'); du = torch.empty((B, H), dtype=torch.float64, device='cuda')
tv, tu = torch.from_numpy(v0), torch.from_numpy(u)
torch.cuda.synchronize(); t = time.perf_counter()
for _ in range(n):
    dv.copy_(tv, non_blocking=True); du.copy_(tu, non_blocking=True)
torch.cuda.synchronize()
print("H2D 713 KB (2 copies) us/step %.1f" % ((time.perf_counter() - t) / n * 1e6))
t = time.perf_counter()
lib = F._lib.load()
for _ in range(n): lib.b2n_version()
print("ctypes call overhead us %.2f" % ((time.perf_counter() - t) / n * 1e6))
# component timings of the public call
rbm.stage(v0, u); torch.cuda.synchronize()
t = time.perf_counter()
for _ in range(n): rbm.stage(v0, u)
print("stage (H2D + sync) us %.1f" % ((time.perf_counter() - t) / n * 1e6))
t = time.perf_counter()
for _ in range(n):
    rbm.run_staged(1, 0.1, B); rbm.recon()
print("run_staged + recon (launch, D2H, sync) us %.1f" % ((time.perf_counter() - t) / n * 1e6))
