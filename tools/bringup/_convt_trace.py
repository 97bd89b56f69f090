# bring-up: per-tile role timeline (CTA 0, clock64) of the halo-tile conv kernels of one ImageNet-shape step
import ctypes as C, numpy as np, os, sys
os.environ["B2N_TRACE"] = "1"
sys.path.insert(0, '.')
from paper_1804_04512_b200 import _lib, fastnn as F, configs as CF
lib = _lib.load()
lib.b2n_debug_trace_read.argtypes = [C.c_void_p, C.c_longlong, C.POINTER(C.c_int)]
spec = CF.NET_CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "imagenet_cnn"]()
net = F.build_network(spec)
B = spec["batch_size"]
x = np.random.default_rng(1).random((B, *spec["input"]), dtype=np.float32)
lab = np.arange(B, dtype=np.int32) % 10
net.stage(x, lab)
net.run_staged(1, B)
buf = np.zeros(64 * 512 * 64, np.uint64); reg = C.c_int()
lib.b2n_debug_trace_read(buf.ctypes.data_as(C.c_void_p), buf.size, C.byref(reg))
names = ["prod", "landed", "split", "mma0", "mma1", "epi0", "epi1"]
for r in range(reg.value):
    t = buf[r * 512 * 64: r * 512 * 64 + 512].astype(np.int64).reshape(64, 8)[:, :7]
    if not t.any(): continue
    t0 = t[t > 0].min()
    rel = np.where(t > 0, t - t0, -1)
    n = int((t[:, 3] > 0).sum())
    print(f"region {r}: tiles traced {n}")
    for it in list(range(min(n, 6))) + list(range(max(6, n - 3), n)):
        print("   tile %2d: " % it + " ".join("%s=%7d" % (names[e], rel[it, e]) for e in range(7)))
    if n > 8:
        d = lambda a, b: np.median(t[4:n, b] - t[4:n, a])
        per = np.median(np.diff(t[4:n, 3]))
        print("   steady: tile period %.0f clk | split %.0f | mma issue %.0f | epi %.0f | land->mma %.0f | mma->epi %.0f" % (
            per, d(1, 2), d(3, 4), d(5, 6), d(1, 3), d(4, 5)))
