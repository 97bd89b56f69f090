import ctypes as C, numpy as np, torch, sys
sys.path.insert(0, '.')
from paper_1804_04512_b200 import _lib
lib = _lib.load()
lib.b2n_debug_probe.argtypes = [C.c_void_p, C.c_longlong, C.c_int, C.c_void_p, C.c_longlong, C.c_int, C.c_void_p, C.c_void_p]
A = np.zeros((128, 32), np.float32); B = np.zeros((32, 32), np.float32)
vals = [1 + 2**-11 + 2**-12, 1 + 2**-11, 1 + 2**-12, -(1 + 2**-11 + 2**-12), 1 + 2**-10 + 2**-11, 3.0000001]
for i, v in enumerate(vals): A[i, 0] = v
B[0, 0] = 1.0
Ad = torch.from_numpy(A).cuda(); Bd = torch.from_numpy(B).cuda()
sm = torch.zeros(5120, device='cuda'); d = torch.zeros(128*32, device='cuda')
lib.b2n_debug_probe(Ad.data_ptr(), 32, 0, Bd.data_ptr(), 32, 0, sm.data_ptr(), d.data_ptr())
d = d.cpu().numpy().reshape(128, 32)
for i, v in enumerate(vals):
    x = np.float32(v); bits = x.view(np.uint32)
    trunc = np.uint32(bits & 0xFFFFE000).view(np.float32)
    print(f"x={float(x)!r:25} hw={float(d[i,0])!r:25} trunc={float(trunc)!r:25} {'TRUNC' if d[i,0]==trunc else 'ROUND/OTHER'}")
