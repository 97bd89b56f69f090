# bring-up: phase timeline of the one-launch CRBM CD-1 kernel (B2N_TRACE=1, %globaltimer ns)
import ctypes as C, os, sys
os.environ["B2N_TRACE"] = "1"
sys.path.insert(0, '.')
import numpy as np
from oracle import oracle as O
from paper_1804_04512_b200 import fastnn as F, _lib
lib = _lib.load()
c, h, w, k, kh, kw, B = 1, 28, 28, 12, 5, 5, 100
m = F.Crbm(c, h, w, k, kh, kw); m.init(42)
m.stage(O.bernoulli_f32(3, 0.5, B * 784).reshape(B, 1, 28, 28), O.canonical_f64(5, B * k * 576))
m.run_staged(20, 0.1, B)
buf = np.zeros(64 * 512 * 64, np.uint64)
n = C.c_int()
lib.b2n_debug_trace_read(buf.ctypes.data_as(C.c_void_p), C.c_longlong(buf.size), C.byref(n))
t = buf[:B * 64].reshape(B, 64)[:, :10].astype(np.int64)
t0 = t[:, 0].min()
names = ["start", "P", "load", "p1", "p2", "p3", "p4", "ticket", "staged", "end"]
for nm, col in zip(names, t.T):
    v = col[col > 0]
    if len(v):
        print("%-7s med %7.2f  min %7.2f  max %7.2f us" % (nm, np.median(v - t0) / 1e3, (v.min() - t0) / 1e3, (v.max() - t0) / 1e3))
