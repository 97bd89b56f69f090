"""The NCCL data-parallel step path on the GPU with a 1-rank communicator (the only GPU count this
environment provides): forward_backward -> ncclAllReduce(packed grads) -> packed SGD kernel must
equal the fused single-GPU step; the same for the RBM (allreduce + W += lr/B dW)."""
import numpy as np
import pytest

from conftest import norm_err
from oracle import oracle as O
from paper_1804_04512_b200 import configs as CF

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("name", ["mlp", "mnist_cnn"])
def test_nccl_step_matches_fused(gpu, name):
    from paper_1804_04512_b200 import fastnn as F
    spec = CF.NET_CONFIGS[name](50)
    x = O.uniform_f32(1, 50 * int(np.prod(spec["input"]))).reshape([50] + spec["input"])
    lab = O.uniform_int(2, 0, 9, 50)
    a = F.build_network(spec)
    b = F.build_network(spec)
    b.dp_init(F.nccl_unique_id(), 0, 1)
    for _ in range(2):
        F.train_minibatch_labels(a, x, lab)
        b.forward_backward(x, lab, 50)
        b.apply_update()
    for i in range(a.num_params()):
        assert norm_err(b.get_param(i), a.get_param(i)) < 1e-6
    b.stage(x, lab)
    b.run_staged(3, 50)  # graph-captured split step: forward/backward, allreduce, SGD
    assert np.isfinite(b.loss())


def test_nccl_rbm_matches_single(gpu):
    from paper_1804_04512_b200 import fastnn as F
    v0 = O.bernoulli_f32(3, 0.5, 100 * 784).reshape(100, 784)
    u = O.canonical_f64(5, 100 * 500).reshape(100, 500)
    a = F.Rbm(500, 784)
    a.init(42)
    b = F.Rbm(500, 784)
    b.init(42)
    b.dp_init(F.nccl_unique_id(), 0, 1)
    a.stage(v0, u)
    b.stage(v0, u)
    a.run_staged(2, 0.1, 100)
    b.run_staged(2, 0.1, 100)
    wa, bva, bha = a.get()
    wb, bvb, bhb = b.get()
    # both run the fused CD-1 kernel; in data-parallel mode it stores the raw sums, NCCL sums them over
    # the ranks and one axpy applies lr / B_global -- the same products, so agreement to rounding
    assert b.kernels_per_step() == 2 and a.kernels_per_step() == 1
    assert norm_err(wb, wa) < 1e-6 and norm_err(bvb, bva) < 1e-6 and norm_err(bhb, bha) < 1e-6
    assert abs(a.recon() - b.recon()) < 1e-6 * a.recon()


def test_nccl_crbm_matches_single(gpu):
    """the data-parallel CRBM step (shard sums -> ncclAllReduce -> update) on a 1-rank communicator
    equals the single-GPU one-launch step"""
    from paper_1804_04512_b200 import fastnn as F
    c, h, w, k, kh, kw, B = 1, 28, 28, 12, 5, 5, 40
    v0 = O.bernoulli_f32(3, 0.5, B * c * h * w).reshape(B, c, h, w)
    u = O.canonical_f64(5, B * k * 24 * 24)
    a, b = F.Crbm(c, h, w, k, kh, kw), F.Crbm(c, h, w, k, kh, kw)
    a.init(42)
    b.init(42)
    b.dp_init(F.nccl_unique_id(), 0, 1)
    for _ in range(2):
        ra = F.crbm_cd_update(a, v0, 0.1, u)
        rb = F.crbm_cd_update(b, v0, 0.1, u, batch_global=B)
        assert abs(ra - rb) <= 1e-9 * ra
    assert b.kernels_per_step() == 2
    for x, y in zip(a.get(), b.get()):
        assert norm_err(y, x) < 1e-6
