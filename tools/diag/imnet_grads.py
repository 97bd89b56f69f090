"""Diagnostic: ImageNet-shape gradients (forward_backward, no update) of the B200 path vs the
restatement in exact-sum mode and vs the reference, at several batch sizes."""
import sys, time
import numpy as np
sys.path.insert(0, "/root/repo"); sys.path.insert(0, "/root/repo/tests")
from conftest import norm_err
from oracle import oracle as O
from paper_1804_04512_b200 import configs as CF
from paper_1804_04512_b200 import fastnn as F

for B in [int(a) for a in sys.argv[1:]] or [16, 128]:
    spec = CF.imagenet_cnn_spec(B)
    x = O.uniform_f32(1, B * 3 * 256 * 256).reshape(B, 3, 256, 256)
    lab = O.uniform_int(2, 0, 999, B)
    net = F.build_network(spec)
    lg = net.forward_backward(x, lab)
    O.set_exact_sums(True)
    ex = O.Net(spec, "oracle"); le = ex.forward_backward(x, lab)
    O.set_exact_sums(False)
    rf = O.Net(spec, "oracle"); lr_ = rf.forward_backward(x, lab)
    print(f"B={B} loss gpu {lg} ref {lr_} exact {le}")
    for i in range(net.num_params()):
        g = net.get_param(i, F.GRAD).ravel()
        e, r = ex.get(i, 1), rf.get(i, 1)
        k = int(np.argmax(np.abs(g.astype(np.float64) - e)))
        print(f"  p{i:2d} n={g.size:8d} gpu-vs-exact {norm_err(g, e):.3e} ref-vs-exact {norm_err(r, e):.3e} "
              f"gpu-vs-ref {norm_err(g, r):.3e}  worst[{k}] gpu {g[k]:.6e} exact {e[k]:.6e} ref {r[k]:.6e}", flush=True)
