import ctypes as C, numpy as np, torch, sys
sys.path.insert(0, '.')
from paper_1804_04512_b200 import _lib
lib = _lib.load()
lib.b2n_debug_gemm_trace.argtypes = [C.c_void_p, C.c_longlong, C.c_int, C.c_void_p, C.c_longlong, C.c_int, C.c_void_p, C.c_longlong, C.c_longlong, C.c_longlong, C.c_longlong, C.c_int, C.c_int, C.c_void_p, C.POINTER(C.c_int)]
for (M, N, K, ta, tb) in [(100, 500, 784, 0, 1), (100, 784, 500, 0, 0), (501, 785, 200, 1, 0), (100, 250, 500, 0, 1)]:
  for prec in (0, 1):
    A = torch.randn((K, M) if ta else (M, K), device='cuda'); B = torch.randn((N, K) if tb else (K, N), device='cuda')
    A = torch.nn.functional.pad(A, (0, (-A.shape[1]) % 8)); B = torch.nn.functional.pad(B, (0, (-B.shape[1]) % 8))
    Cm = torch.zeros(M, N, device='cuda')
    tr = torch.zeros(1024 * 64, dtype=torch.int64, device='cuda'); g = C.c_int()
    for rep in range(3):
        st = lib.b2n_debug_gemm_trace(A.data_ptr(), A.stride(0), ta, B.data_ptr(), B.stride(0), tb, Cm.data_ptr(), N, M, N, K, prec, 0, tr.data_ptr(), C.byref(g))
    assert st == 0, lib.b2n_last_error()
    a = A[:, :(M if ta else K)]; b = B[:, :(K if tb else N)]
    ref = (a.T if ta else a).double() @ (b.T if tb else b).double()
    err = (Cm.double() - ref).abs().max().item() / ref.abs().max().item()
    t = tr.cpu().numpy().reshape(-1, 64)[:g.value].astype(np.float64)
    t0 = t[:, 0].min(); r = (t - t0) / 1000.0
    b0 = r[0]
    print(f"M={M} N={N} K={K} {'x3' if prec==0 else 'x1'} ctas={g.value} span {r[:,52].max():.2f}us err {err:.1e} start spread {r[:,0].max():.2f}")
    nk = int(np.sum(b0[34:50] > -1e6))
    print("   b0: setup %.2f | tma %s | landed %s | mma %s | commit %.2f tile %.2f part %.2f cbar %.2f red %.2f epi %.2f end %.2f" % (
        b0[1], " ".join("%.2f" % x for x in b0[2:2+min(nk,8)]), " ".join("%.2f" % x for x in b0[18:18+min(nk,8)]),
        " ".join("%.2f" % x for x in b0[34:34+min(nk,8)]), b0[50], b0[53], b0[54], b0[55], b0[56], b0[57], b0[52]))
    print("   median over CTAs: commit %.2f tile %.2f part %.2f cbar %.2f red %.2f epi %.2f end %.2f" % tuple(np.median(r[:, i]) for i in (50, 53, 54, 55, 56, 57, 52)))
