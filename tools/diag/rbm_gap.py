"""Inter-step gap of the streamed fused CD-1 step (B2N_RBM_TRACE=1): step i's last CTA exit, step i+1's
first CTA entry / first CTA past griddepcontrol.wait + the readiness poll, from %globaltimer."""
import ctypes as C
import os
import sys
os.environ["B2N_RBM_TRACE"] = "1"
sys.path.insert(0, ".")
import numpy as np
import torch
from paper_1804_04512_b200 import fastnn as F, _lib

lib = _lib.load()
B, H, V = 100, 500, 784
r = F.Rbm(H, V)
r.init(1)
dev = torch.device("cuda", 0)
for K in (2, 3, 6, 7):
    v = (torch.rand(K * B, V, device=dev) < 0.5).float()
    u = torch.rand(K * B, H, device=dev, dtype=torch.float64)
    r.train_stream_ptr(v.data_ptr(), u.data_ptr(), K, B, 0.1)
    buf = np.zeros(512, np.uint64)
    lib.b2n_debug_rbm_trace(r.handle, buf.ctypes.data_as(C.c_void_p))
    last = (K - 1) & 1
    a, b = buf[256 * (1 - last):256 * (2 - last)].astype(np.int64), buf[256 * last:256 * (last + 1)].astype(np.int64)
    ea, fa, xa = a[64:128], a[128:192], a[192:256]
    eb, fb, xb = b[64:128], b[128:192], b[192:256]
    t0 = ea.min()
    us = lambda x: (x - t0) / 1e3
    print(f"K={K}: step n-1 entry {us(ea.min()):.2f}..{us(ea.max()):.2f} waited {us(fa.min()):.2f}..{us(fa.max()):.2f} "
          f"exit {us(xa.min()):.2f}..{us(xa.max()):.2f} | step n entry {us(eb.min()):.2f}..{us(eb.max()):.2f} "
          f"waited {us(fb.min()):.2f}..{us(fb.max()):.2f} exit {us(xb.min()):.2f}..{us(xb.max()):.2f}")
