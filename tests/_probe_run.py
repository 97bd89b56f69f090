import ctypes as C, numpy as np, torch, sys
sys.path.insert(0, '.')
from paper_1804_04512_b200 import _lib
lib = _lib.load()
lib.b2n_debug_probe.argtypes = [C.c_void_p, C.c_longlong, C.c_int, C.c_void_p, C.c_longlong, C.c_int, C.c_void_p, C.c_void_p]
def swz_k(tile):  # expected SW128 K-major layout of a rows x 32 fp32 tile
    rows = tile.shape[0]
    out = np.zeros(rows * 32, np.float32)
    for m in range(rows):
        for k in range(32):
            off = (m // 8) * 1024 + (m % 8) * 128 + (((k // 4) ^ (m % 8)) * 16) + (k % 4) * 4
            out[off // 4] = tile[m, k]
    return out
for a_mn, b_mn in [(0,0),(1,0),(0,1),(1,1)]:
    rng = np.random.default_rng(0)
    A = rng.integers(-3, 4, (128, 32)).astype(np.float32)   # logical M x K
    B = rng.integers(-3, 4, (32, 32)).astype(np.float32)    # logical N x K
    Ad = torch.from_numpy(np.ascontiguousarray(A.T if a_mn else A)).cuda()
    Bd = torch.from_numpy(np.ascontiguousarray(B.T if b_mn else B)).cuda()
    sm = torch.zeros(5120, device='cuda'); d = torch.zeros(128*32, device='cuda')
    st = lib.b2n_debug_probe(Ad.data_ptr(), Ad.stride(0), a_mn, Bd.data_ptr(), Bd.stride(0), b_mn, sm.data_ptr(), d.data_ptr())
    print("status", st, lib.b2n_last_error())
    sm = sm.cpu().numpy(); d = d.cpu().numpy().reshape(128, 32)
    want = A @ B.T
    if not a_mn:
        print("A smem matches SW128 K-major:", np.array_equal(sm[:4096], swz_k(A)), "nonzero", np.count_nonzero(sm[:4096]))
    else:
        print("A smem nonzero", np.count_nonzero(sm[:4096]), "first row", sm[:8])
    print(f"a_mn={a_mn} b_mn={b_mn} D max err {np.abs(d-want).max()} nonzero {np.count_nonzero(d)}; D[0,:6]={d[0,:6]} want {want[0,:6]}")
    if np.abs(d-want).max() > 0:
        # try to identify permutations
        print("D == A@B ?", np.abs(d - A @ B).max() if True else None)

# GEMM sweep: localize failures by precision / shape / majors
from paper_1804_04512_b200 import fastnn as F
from oracle import oracle as O
def dev(x):
    r, c = x.shape; cp = (c + 7)//8*8
    t = torch.zeros((r, cp), dtype=torch.float32, device='cuda'); t[:, :c] = torch.from_numpy(x); return t[:, :c]
for (M,N,K) in [(128,32,32),(128,64,32),(128,32,64),(128,32,160),(100,500,784),(256,64,32),(37,53,29)]:
    for ta in (0,1):
        for tb in (0,1):
            rng = np.random.default_rng(1)
            a = rng.integers(-3,4,((K,M) if ta else (M,K))).astype(np.float32)
            b = rng.integers(-3,4,((N,K) if tb else (K,N))).astype(np.float32)
            want = O.gemm(ta,tb,a,b)
            res = []
            for prec in (F.TF32, F.TF32X3):
                got = F.gemm(dev(a), dev(b), bool(ta), bool(tb), precision=prec).cpu().numpy()
                res.append(f"{np.abs(got-want).max():.3g}/{np.count_nonzero(got)}")
            print(f"M={M} N={N} K={K} ta={ta} tb={tb}: x1 {res[0]}  x3 {res[1]}  (nnz want {np.count_nonzero(want)})")
