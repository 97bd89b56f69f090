"""Shape coverage of the halo-tile conv kernels (csrc/convt.cuh) against the oracle restatement of
conv_forward / conv_backward / pool (layers.hpp:132-271): channel counts that are not multiples of 4
(zero-padded quads), 1 / 2 / 3 / 5 quads, pad 0 / 1 / 2, 3x3 and 5x5 filters, up to 32 kernels (the
N = kh * 32 MMA), odd output widths, convs without pooling (the full-resolution epilogue), stacks
whose last conv feeds a dense layer in NCHW order, and a 7x7 net that takes the implicit-GEMM
fallback (csrc/conv.cuh) because it is outside the halo-tile envelope. Gradients after one forward/backward within 1e-4
(normalised), parameters after two SGD steps within 1e-3 -- the 3xTF32 contract of DESIGN.md 4."""
import numpy as np
import pytest

from conftest import norm_err
from oracle import oracle as O
from paper_1804_04512_b200 import configs as CF

pytestmark = pytest.mark.gpu


def spec_of(inp, convs, batch, act, dense_out=10):
    """convs: list of (k, kh, pad, pool)."""
    c, h, w = inp
    layers = []
    for k, kh, pad, pool in convs:
        layers += [CF.conv(k, kh, kh, pad), act()]
        h, w, c = h + 2 * pad - kh + 1, w + 2 * pad - kh + 1, k
        if pool:
            layers.append(CF.maxpool())
            h, w = h // 2, w // 2
    layers += [CF.dense(c * h * w, dense_out), CF.softmax()]
    return {"name": "convt_shape", "input": list(inp), "layers": layers, "lr": 0.05, "momentum": 0.9,
            "weight_decay": 0.0, "batch_size": batch, "seed": 7}


CASES = [
    # (input, convs, batch, act)
    ((5, 16, 16), [(6, 3, 1, True), (10, 3, 1, True)], 3, CF.relu),        # C = 5, 6 (2 quads), K = 10
    ((2, 20, 18), [(12, 5, 2, True), (7, 3, 0, False)], 2, CF.sigmoid),   # pad 2, 5x5, no pool
    ((3, 20, 20), [(6, 7, 0, True)], 2, CF.relu),                         # 7x7: the implicit-GEMM fallback
    ((16, 12, 12), [(32, 3, 1, True)], 4, CF.relu),                       # 4 quads -> 32 kernels
    ((1, 17, 17), [(9, 3, 0, False), (4, 5, 1, False)], 2, CF.sigmoid),   # odd widths, 1 channel
    ((3, 36, 36), [(12, 5, 0, True), (12, 5, 0, True)], 2, CF.relu),      # CIFAR-like, 3 quads
    ((4, 14, 10), [(8, 3, 1, True), (16, 3, 1, False)], 3, CF.relu),      # pooled maps of odd extent (7x5)
    ((3, 64, 64), [(16, 3, 1, True), (16, 3, 1, True)], 2, CF.sigmoid),   # ImageNet-like 3x3 pad 1, tall tiles
]


@pytest.mark.parametrize("case", range(len(CASES)))
def test_convt_shape(gpu, case):
    from paper_1804_04512_b200 import fastnn as F
    inp, convs, B, act = CASES[case]
    spec = spec_of(inp, convs, B, act)
    net = F.build_network(spec)
    orc = O.Net(spec)
    per = int(np.prod(inp))
    x = O.uniform_f32(11 + case, B * per).reshape([B] + list(inp))
    lab = O.uniform_int(3, 0, 9, B)
    lg = net.forward_backward(x, lab)
    lo = orc.forward_backward(x, lab)
    assert abs(lg - lo) <= 1e-5 * abs(lo), (lg, lo)
    for i in range(net.num_params()):
        assert norm_err(net.get_param(i, F.GRAD).ravel(), orc.get(i, 1)) < 1e-4, i
    net2 = F.build_network(spec)
    orc2 = O.Net(spec)
    for _ in range(2):
        F.train_minibatch_labels(net2, x, lab)
        orc2.train_minibatch(x, lab)
    for i in range(net2.num_params()):
        assert norm_err(net2.get_param(i).ravel(), orc2.get(i)) < 1e-3, i


def test_fused_rbm_matches_split_path(gpu, monkeypatch):
    """The fused single-kernel CD-1 step (rbm_fused.cuh) and the 4-GEMM split path (B2N_RBM_FUSED=0)
    compute the same step: identical samples on these inputs, parameters / states within 3xTF32."""
    from paper_1804_04512_b200 import fastnn as F
    B, H, V = 100, 500, 784
    v0 = O.bernoulli_f32(3, 0.5, B * V).reshape(B, V)
    u = O.canonical_f64(5, B * H).reshape(B, H)
    a = F.Rbm(H, V)
    a.init(42)
    ra = F.cd_k_update(a, v0, 1, 0.1, u)
    monkeypatch.setenv("B2N_RBM_FUSED", "0")
    b = F.Rbm(H, V)
    b.init(42)
    rb = F.cd_k_update(b, v0, 1, 0.1, u)
    assert a.kernels_per_step() == 1 and b.kernels_per_step() == 4
    sa, sb = a.last_states(B), b.last_states(B)
    for x, y in zip(sa, sb):
        assert norm_err(x, y) < 1e-5
    np.testing.assert_array_equal(sa[1], sb[1])  # samples
    for x, y in zip(a.get(), b.get()):
        assert norm_err(x, y) < 1e-5
    assert abs(ra - rb) < 1e-6 * abs(rb)
