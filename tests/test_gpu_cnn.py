"""CNN training steps (configs 3-5) on the B200 vs the oracle restatement of train_minibatch with
conv_forward / conv_backward / pool (layers.hpp:132-271). Tolerance as for the MLP: 3xTF32
implicit-GEMM convs -> normalized error <= 1e-4 on loss, <= 1e-3 on every updated parameter."""
import numpy as np
import pytest

from conftest import check_argmax, norm_err
from oracle import oracle as O
from paper_1804_04512_b200 import configs as CF

pytestmark = pytest.mark.gpu


def small_imagenet(batch=2, hw=32):
    spec = CF.imagenet_cnn_spec(batch, hw)
    side = hw // 32
    spec["layers"][-4] = CF.dense(16 * side * side, 64)
    spec["layers"][-2] = CF.dense(64, 100)
    return spec


def run_steps(spec, B, steps=2, tol_p=1e-3, x=None, which="oracle"):
    from paper_1804_04512_b200 import fastnn as F
    net = F.build_network(spec)
    orc = O.Net(spec, which)
    for i in range(net.num_params()):
        np.testing.assert_array_equal(net.get_param(i).ravel(), orc.get(i))
    per = int(np.prod(spec["input"]))
    classes = [d for d in spec["layers"] if d["kind"] == CF.DENSE][-1]["out"]
    if x is None:
        x = O.uniform_f32(1, B * per).reshape([B] + spec["input"])
    lab = O.uniform_int(2, 0, classes - 1, B)
    for step in range(steps):
        lg = F.train_minibatch_labels(net, x, lab)
        lo = orc.train_minibatch(x, lab)
        assert abs(lg - lo) <= 1e-4 * abs(lo), (step, lg, lo)
        for i in range(net.num_params()):
            e = norm_err(net.get_param(i).ravel(), orc.get(i))
            assert e < tol_p, (step, i, e)
    return net, orc


@pytest.mark.parametrize("B", [100, 7, 1])
def test_mnist_cnn_step(gpu, B):
    run_steps(CF.mnist_cnn_spec(B), B)


@pytest.mark.parametrize("B", [100, 3])
def test_cifar_cnn_step(gpu, B):
    run_steps(CF.cifar_cnn_spec(B), B)


def test_imagenet_shape_small_step(gpu):
    """pad=1 convs: the backward is the SURVEY 8(c) composite (parity unpinned by the reference's
    own tests; the oracle composite is bit-exact with reference primitives, see test_oracle)."""
    run_steps(small_imagenet(2, 32), 2)


@pytest.mark.parametrize("B", [16, 128])
def test_imagenet_cnn_baseline_shape(gpu, B):
    """BASELINE config 5 at its real shape: 3x256x256 input, five conv(16, 3x3, pad 1) + relu +
    2x2 pool blocks, dense 1024 -> 2048 relu -> 1000 softmax (layers.hpp:132-320, network.hpp:410-437).
    B = 16 is the 8-GPU shard, B = 128 the whole global batch. This runs the 256^2 / 128^2 halo-tile
    plans, the wgrad run lengths and the > 256-class softmax_xent_rows_kernel. The checker is the
    SURVEY 8(c) composite of reference primitives: the reference compiled from its headers
    (oracle/_ref, multithreaded, bitwise independent of the thread count) when present, else the
    scalar restatement (bit-identical to it, tests/test_oracle.py)."""
    import os
    which = "ref" if O.ref_available() else "oracle"
    if which == "ref":
        O.load("ref").ref_set_threads(os.cpu_count() or 1)
    elif B > 16:
        pytest.skip("the scalar restatement takes minutes at B = 128; needs oracle/_ref")
    from paper_1804_04512_b200 import fastnn as F
    spec = CF.imagenet_cnn_spec(B)
    x = O.uniform_f32(1, B * 3 * 256 * 256).reshape(B, 3, 256, 256)
    net, orc = run_steps(spec, B, steps=2 if B == 16 else 1, x=x, which=which)
    # inference on the updated parameters: 1000-class probabilities and first-max argmax
    probs, am = F.forward_batch(net, x, return_argmax=True)
    op, oa = orc.forward(x)
    assert norm_err(probs, op) < 1e-4
    check_argmax(am, probs, op, oa, max_near_frac=0.05)


def test_mlp_argmax_dataset_scale(gpu):
    """argmax over 4000 inputs on trained parameters (forward_batch, network.hpp:402 + :66-72):
    the near-tie count is reported and bounded"""
    from paper_1804_04512_b200 import fastnn as F
    spec = CF.mlp_spec(100)
    net = F.build_network(spec)
    orc = O.Net(spec)
    x = O.uniform_f32(21, 4000 * 784).reshape(4000, 784)
    lab = O.uniform_int(22, 0, 9, 4000)
    for i in range(5):
        F.train_minibatch_labels(net, x[100 * i:100 * (i + 1)], lab[100 * i:100 * (i + 1)])
    for i in range(net.num_params()):
        orc.set(i, net.get_param(i).ravel())
    probs, am = F.forward_batch(net, x, return_argmax=True)
    op, oa = orc.forward(x)
    assert norm_err(probs, op) < 1e-5
    check_argmax(am, probs, op, oa, max_near_frac=0.002)


def test_cnn_grads(gpu):
    from paper_1804_04512_b200 import fastnn as F
    spec = CF.mnist_cnn_spec(20)
    net = F.build_network(spec)
    orc = O.Net(spec)
    x = O.uniform_f32(1, 20 * 784).reshape(20, 1, 28, 28)
    lab = O.uniform_int(2, 0, 9, 20)
    lg = net.forward_backward(x, lab)
    lo = orc.forward_backward(x, lab)
    assert abs(lg - lo) <= 1e-5 * lo
    for i in range(net.num_params()):
        assert norm_err(net.get_param(i, F.GRAD).ravel(), orc.get(i, 1)) < 1e-4, i


def test_pool_ties_first_index(gpu):
    """layers.hpp:228-232 / test_layers.cpp pooling ties: relu zeros tie, the first index wins,
    and the routed gradient goes to that first position (all-negative pre-activations)."""
    from paper_1804_04512_b200 import fastnn as F
    spec = CF.cifar_cnn_spec(4)
    net = F.build_network(spec)
    orc = O.Net(spec)
    # large negative first-layer bias -> relu outputs all zero -> every pooling window ties
    b = net.get_param(1)
    b[:] = -50.0
    net.set_param(1, b)
    orc.set(1, b)
    x = O.uniform_f32(3, 4 * 3 * 32 * 32).reshape(4, 3, 32, 32)
    lab = O.uniform_int(4, 0, 9, 4)
    lg = net.forward_backward(x, lab)
    lo = orc.forward_backward(x, lab)
    assert abs(lg - lo) <= 1e-5 * lo
    for i in range(net.num_params()):
        assert norm_err(net.get_param(i, F.GRAD).ravel(), orc.get(i, 1)) < 1e-4, i
