"""Diagnostic: per-layer forward of the ImageNet-shape CNN (pooled outputs + argmax codes) vs the
reference's conv_forward (oracle restatement, bit-exact with it) + relu + first-index 2x2 max."""
import sys
import numpy as np
sys.path.insert(0, "/root/repo")
from oracle import oracle as O
from paper_1804_04512_b200 import configs as CF
from paper_1804_04512_b200 import fastnn as F


def pool_ref(a):
    n, k, h, w = a.shape
    win = a.reshape(n, k, h // 2, 2, w // 2, 2).transpose(0, 1, 2, 4, 3, 5).reshape(n, k, h // 2, w // 2, 4)
    code = np.zeros(win.shape[:-1], np.uint8)
    best = win[..., 0].copy()
    for i in range(1, 4):
        m = win[..., i] > best
        best[m] = win[..., i][m]
        code[m] = i
    return best, code


B = int(sys.argv[1]) if len(sys.argv) > 1 else 128
spec = CF.imagenet_cnn_spec(B)
net = F.build_network(spec)
x = O.uniform_f32(1, B * 3 * 256 * 256).reshape(B, 3, 256, 256)
lab = O.uniform_int(2, 0, 999, B)
net.forward_backward(x, lab)
cur = x
for L in range(5):
    K = net.get_param(2 * L).reshape(16, -1, 3, 3)
    b = net.get_param(2 * L + 1)
    z = O.conv_forward(cur, K, b, pad=1)
    ref, rc = pool_ref(np.maximum(z, 0))
    got, gc = net.layer_output(L, B, ref.shape[1:])
    d = np.abs(got.astype(np.float64) - ref)
    bad = np.argwhere(gc != rc)
    print(f"conv{L}: max|dP| {d.max():.3e} (rel {d.max() / np.abs(ref).max():.2e}), code mismatches {len(bad)} / {gc.size}")
    for idx in bad[:6]:
        bb, kk, yy, xx = idx
        zw = z[bb, kk, 2 * yy:2 * yy + 2, 2 * xx:2 * xx + 2].ravel()
        print(f"   at {tuple(idx)} gpu code {gc[tuple(idx)]} ref {rc[tuple(idx)]} gpuP {got[tuple(idx)]:.7e} refP {ref[tuple(idx)]:.7e} z {zw}")
    cur = ref  # continue from the reference's activations
