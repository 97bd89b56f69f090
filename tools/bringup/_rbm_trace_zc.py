# bring-up: fused CD-1 phase timeline, staged (device inputs) vs zero-copy (pinned host inputs)
import ctypes as C, os, sys
os.environ["B2N_RBM_TRACE"] = "1"
sys.path.insert(0, '.')
import numpy as np, torch
from oracle import oracle as O
from paper_1804_04512_b200 import fastnn as F, _lib
lib = _lib.load()
B, V, H = 100, 784, 500
v0 = torch.empty((B, V), dtype=torch.float32, pin_memory=True).numpy(); v0[:] = O.bernoulli_f32(3, 0.5, B * V).reshape(B, V)
u = torch.empty((B, H), dtype=torch.float64, pin_memory=True).numpy(); u[:] = O.canonical_f64(5, B * H).reshape(B, H)
names = ["start", "p1.mma", "p1.cbar", "p1.red", "p1.end", "bar1", "p2.mma", "p2.wr", "bar2", "p2.red", "bar3",
         "p3.mma", "p3.cbar", "p3.red", "p3.end", "bar4", "p4.mma", "p4.end"]
for mode in ("staged", "zero-copy", "zero-copy"):
    rbm = F.Rbm(H, V); rbm.init(42)
    if mode == "staged":
        rbm.stage(np.array(v0), np.array(u)); rbm.run_staged(3, 0.1, B)
    else:
        for _ in range(3): F.cd_k_update(rbm, v0, 1, 0.1, u)
    buf = np.zeros(256, np.uint64)
    lib.b2n_debug_rbm_trace(rbm.handle, buf.ctypes.data_as(C.c_void_p))
    print(mode)
    for base in (0, 32):
        t = buf[base:base + len(names)].astype(np.int64)
        print("  " + " ".join("%s=%.2f" % (n, (x - t[0]) / 1965.0) for n, x in zip(names, t)))
    e, f, x = buf[64:128].astype(np.int64), buf[128:192].astype(np.int64), buf[192:256].astype(np.int64)
    t0 = e.min()
    print("  entry skew %.2f us, end med %.2f max %.2f us" % ((e.max() - t0) / 1e3, np.median(x - t0) / 1e3, (x.max() - t0) / 1e3))
