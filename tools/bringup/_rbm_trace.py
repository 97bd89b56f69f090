# bring-up: phase timeline of the fused CD-1 kernel (CTA (0,0) and (7,7), clock64 -> us at 1.965 GHz)
import ctypes as C, os, sys
os.environ["B2N_RBM_TRACE"] = "1"
sys.path.insert(0, '.')
import numpy as np
from oracle import oracle as O
from paper_1804_04512_b200 import fastnn as F, _lib
lib = _lib.load()
rbm = F.Rbm(500, 784); rbm.init(42)
rbm.stage(O.bernoulli_f32(3, 0.5, 100 * 784).reshape(100, 784), O.canonical_f64(5, 100 * 500).reshape(100, 500))
rbm.run_staged(5, 0.1, 100)
buf = np.zeros(512, np.uint64)
lib.b2n_debug_rbm_trace(rbm.handle, buf.ctypes.data_as(C.c_void_p))
names = ["start", "p1.mma", "p1.cbar", "p1.red", "p1.end", "bar1", "p2.mma", "p2.wr", "bar2", "p2.red", "bar3",
         "p3.mma", "p3.cbar", "p3.red", "p3.end", "bar4", "p4.mma", "p4.ts", "p4.end"]
for base in (0, 32):
    t = buf[base:base + len(names)].astype(np.int64)
    t0 = t[0]
    print(("cta(0,0)" if base == 0 else "cta(7,7)") + " " + " ".join("%s=%.2f" % (n, (x - t0) / 1965.0) for n, x in zip(names, t)))
e, f, x = buf[64:128].astype(np.int64), buf[128:192].astype(np.int64), buf[192:256].astype(np.int64)
t0 = e.min()
print("entry skew us: min 0 max %.2f | setup (entry->first mark) med %.2f max %.2f | end med %.2f max %.2f" % (
    (e.max() - t0) / 1e3, np.median(f - e) / 1e3, (f - e).max() / 1e3, np.median(x - t0) / 1e3, (x.max() - t0) / 1e3))
