import ctypes as C, numpy as np, sys, os, torch
sys.path.insert(0, '.')
os.environ["B2N_TRACE"] = "1"
from paper_1804_04512_b200 import _lib, fastnn as F, configs as CF
from oracle import oracle as O
lib = _lib.load()
lib.b2n_debug_trace_read.argtypes = [C.c_void_p, C.c_longlong, C.POINTER(C.c_int)]
which = sys.argv[1] if len(sys.argv) > 1 else "rbm"
if which == "rbm":
    obj = F.Rbm(500, 784); obj.init(42)
    obj.stage(O.bernoulli_f32(3, 0.5, 100*784).reshape(100, 784), O.canonical_f64(5, 100*500).reshape(100, 500))
    run = lambda n: obj.run_staged(n, 0.1, 100)
else:
    spec = CF.NET_CONFIGS[which](); obj = F.build_network(spec)
    x = O.uniform_f32(1, 100*int(np.prod(spec["input"]))).reshape([100]+spec["input"]); lab = O.uniform_int(2, 0, 9, 100)
    obj.stage(x, lab); run = lambda n: obj.run_staged(n, 100)
flush = torch.empty(512 << 18, device='cuda')
for rep in range(3):
    run(1); torch.cuda.synchronize()
flush.zero_(); torch.cuda.synchronize()
run(1); torch.cuda.synchronize()
buf = np.zeros(64 * 512 * 64, np.uint64); reg = C.c_int()
lib.b2n_debug_trace_read(buf.ctypes.data_as(C.c_void_p), buf.size, C.byref(reg))
t = buf.reshape(64, 512, 64)[:reg.value].astype(np.float64)
valid = t[:, :, 0] > 0
t0 = t[:, :, 0][valid].min()
for i in range(reg.value):
    v = valid[i]
    if not v.any(): continue
    r = (t[i][v] - t0) / 1000.0
    start, end = r[:, 0], r[:, 52]
    print(f"   detail: red_done {np.median(r[:,58]):6.2f} red_sync {np.median(r[:,56]):6.2f} epi_start {np.median(r[:,59]):6.2f} epi_loop_done {np.median(r[:,60]):6.2f}")
    print(f"gemm{i}: ctas {v.sum():3d} start {start.min():7.2f}..{start.max():7.2f}  setup {np.median(r[:,1]):6.2f} mma0 {np.median(r[:,34]):6.2f} commit {np.median(r[:,50]):6.2f} tile {np.median(r[:,53]):6.2f} cbar {np.median(r[:,55]):6.2f} epi_end {np.median(r[:,57]):6.2f} end {end.max():7.2f}")
