"""The oracle (oracle/fastnn_oracle.cpp) pinned to the reference: bit-exact against the golden
fixtures produced by the unmodified reference (tests/golden/make_golden.py), against the
reference's own known-answer tests, and -- where oracle/_ref is built -- against the reference live."""
import json
from pathlib import Path

import numpy as np
import pytest

from conftest import rel_err
from oracle import oracle as O
from paper_1804_04512_b200 import configs as CF

GOLD = Path(__file__).resolve().parent / "golden"
META = json.loads((GOLD / "meta.json").read_text())


def bitwise(a, b):
    a = np.asarray(a)
    b = np.asarray(b)
    return a.shape == b.shape and np.array_equal(a.view(np.uint32), b.view(np.uint32))


def test_gemm_golden():
    g = np.load(GOLD / "gemm.npz")
    for ta in (0, 1):
        for tb in (0, 1):
            c = O.gemm(ta, tb, g[f"a_{ta}{tb}"], g[f"b_{ta}{tb}"])
            assert bitwise(c, g[f"c_{ta}{tb}"].astype(np.float32)), (ta, tb)


@pytest.mark.parametrize("name", ["mlp_small", "mnist_cnn_small", "cifar_cnn_small", "imagenet_cnn_small"])
def test_network_step_golden(name):
    g = np.load(GOLD / f"{name}.npz")
    spec = META[name]["spec"]
    net = O.Net(spec)
    n = net.num_params()
    for i in range(n):
        assert bitwise(net.get(i), g[f"init{i}"]), ("init", i)
    probs = np.zeros_like(g["probs0"])
    loss0 = net.forward_backward(g["x"], g["labels"], probs=probs)
    assert loss0 == g["losses"][0]
    assert bitwise(probs, g["probs0"])
    for i in range(n):
        assert bitwise(net.get(i, 1), g[f"grad{i}"]), ("grad", i)
    net.apply()
    for k in range(1, len(g["losses"])):
        assert net.train_minibatch(g["x"], g["labels"]) == g["losses"][k]
    for i in range(n):
        assert bitwise(net.get(i), g[f"final{i}"]), ("final", i)
        assert bitwise(net.get(i, 2), g[f"vel{i}"]), ("vel", i)
    p, am = net.forward(g["x"])
    assert bitwise(p, g["probs_final"])
    assert np.array_equal(am, g["argmax_final"])


def test_rbm_cd1_golden():
    """The reference draws Bernoulli samples from its std::mt19937(5); the oracle takes the same
    generate_canonical<double,53> stream as supplied uniforms and must match bit for bit."""
    g = np.load(GOLD / "rbm.npz")
    B, H = g["v0"].shape[0], g["W"].shape[0]
    u = O.canonical_f64(int(g["rng_seed"][0]), B * H).reshape(B, H)
    recon, W1, bv1, bh1, _ = O.rbm_cd1(g["W"], g["bv"], g["bh"], g["v0"], 0.1, u)
    assert bitwise(W1, g["W1"]) and bitwise(bv1, g["bv1"]) and bitwise(bh1, g["bh1"])
    assert recon == g["recon"][0]


def test_rbm_cdk_golden():
    """CD-k for k = 2, 3 (energy.hpp:139-144): the reference's chain resamples hs from every
    intermediate visible mean; the oracle consumes the same mt19937(11 + i) stream as k * B * H
    supplied uniforms and must match bit for bit."""
    g = np.load(GOLD / "rbm_cdk.npz")
    i = 0
    while f"W{i}" in g:
        k, B, H = int(g[f"k{i}"][0]), g[f"v0_{i}"].shape[0], g[f"W{i}"].shape[0]
        u = O.canonical_f64(11 + i, k * B * H)
        recon, W1, bv1, bh1, _ = O.rbm_cdk(g[f"W{i}"], g[f"bv{i}"], g[f"bh{i}"], g[f"v0_{i}"], k, 0.1, u)
        assert bitwise(W1, g[f"W1_{i}"]) and bitwise(bv1, g[f"bv1_{i}"]) and bitwise(bh1, g[f"bh1_{i}"]), i
        assert recon == g[f"recon{i}"][0]
        # k = 1 of the general routine is the CD-1 restatement
        r1, Wa, _, _, _ = O.rbm_cdk(g[f"W{i}"], g[f"bv{i}"], g[f"bh{i}"], g[f"v0_{i}"], 1, 0.1, u[:B * H])
        r2, Wb, _, _, _ = O.rbm_cd1(g[f"W{i}"], g[f"bv{i}"], g[f"bh{i}"], g[f"v0_{i}"], 0.1, u[:B * H].reshape(B, H))
        assert r1 == r2 and bitwise(Wa, Wb)
        i += 1
    assert i == 2


def test_sgd_trace_golden():
    """acceptance.cpp:483-555: the 3-step momentum trace with grads {0.3, -0.2, 0.05}."""
    g = np.load(GOLD / "sgd.npz")
    p = np.array([1.0, 0, 0, 0], np.float32)
    v = np.zeros(4, np.float32)
    lib = O.load()
    for k, gv in enumerate((0.3, -0.2, 0.05)):
        gg = np.array([gv, 0, 0, 0], np.float32)
        lib.orc_sgd_momentum_step(O.fptr(p), O.fptr(v), O.fptr(gg), 4, 0.1, 0.9, 0.0)
        assert p[0] == g["trace"][k]


def test_full_size_checksums():
    """One full-batch step of configs 1-4 (+ the padded composite at batch 2, + RBM CD-1) against
    checksums of the reference's own run: pins the oracle at BASELINE sizes."""
    full = json.loads((GOLD / "full_size.json").read_text())
    for name in ["mlp", "mnist_cnn", "cifar_cnn", "imagenet_cnn"]:
        f = full[name]
        spec = CF.NET_CONFIGS[name](f["batch"])
        B = f["batch"]
        per = int(np.prod(spec["input"]))
        classes = [d for d in spec["layers"] if d["kind"] == CF.DENSE][-1]["out"]
        x = O.uniform_f32(1, B * per).reshape([B] + spec["input"])
        lab = O.uniform_int(2, 0, classes - 1, B)
        net = O.Net(spec)
        assert net.train_minibatch(x, lab) == f["loss"], name
        for i in range(net.num_params()):
            assert float(np.sum(net.get(i).astype(np.float64))) == f["param_sums"][i], (name, i)
    c = CF.RBM
    W = O.rbm_init(c["hidden"], c["visible"], c["seed"])
    v0 = O.bernoulli_f32(3, 0.5, c["batch_size"] * c["visible"]).reshape(c["batch_size"], c["visible"])
    u = O.canonical_f64(5, c["batch_size"] * c["hidden"]).reshape(c["batch_size"], c["hidden"])
    recon, W1, bv1, bh1, _ = O.rbm_cd1(W, np.zeros(c["visible"], np.float32), np.zeros(c["hidden"], np.float32),
                                       v0, c["lr"], u)
    assert recon == full["rbm"]["recon"]
    assert float(np.sum(W1.astype(np.float64))) == full["rbm"]["w_sum"]


# ------------------------------------------------ the reference's own known-answer tests, restated
def test_known_gemm_hand_product():  # test_kernels.cpp:33-41
    c = O.gemm(0, 0, np.array([[1, 2], [3, 4]], np.float32), np.array([[5, 6], [7, 8]], np.float32))
    assert np.array_equal(c, np.array([[19, 22], [43, 50]], np.float32))


def test_known_conv_examples():  # test_conv.cpp:37-52
    x = O.uniform_f32(3, 9, -1, 1).reshape(1, 1, 3, 3)
    ker = np.zeros((1, 1, 3, 3), np.float32)
    ker[0, 0, 1, 1] = 1
    assert rel_err(O.conv_forward(x, ker, np.zeros(1, np.float32), pad=1), x) < 1e-6
    y = O.conv_forward(np.array([1, 2, 3, 4], np.float32).reshape(1, 1, 2, 2),
                       np.array([1, 0, 0, 1], np.float32).reshape(1, 1, 2, 2), np.zeros(1, np.float32))
    assert y[0, 0, 0, 0] == 5.0


def test_known_sgd():  # test_optim.cpp:14-69
    lib = O.load()

    def step(p, v, g, lr, mom, wd):
        lib.orc_sgd_momentum_step(O.fptr(p), O.fptr(v), O.fptr(g), 1, lr, mom, wd)

    p, v, g = np.zeros(1, np.float32), np.zeros(1, np.float32), np.ones(1, np.float32)
    step(p, v, g, 0.1, 0.0, 0.0)
    assert rel_err(p[0], -0.1) < 1e-6
    p, v = np.zeros(1, np.float32), np.zeros(1, np.float32)
    step(p, v, g, 0.1, 0.9, 0.0)
    step(p, v, g, 0.1, 0.9, 0.0)
    assert rel_err(p[0], -0.29) < 1e-6
    p, v = np.array([2.0], np.float32), np.zeros(1, np.float32)
    step(p, v, np.zeros(1, np.float32), 0.1, 0.0, 0.5)
    assert rel_err(p[0], 1.9) < 1e-6


def test_known_xent_uniform_is_ln10():  # test_network.cpp:210-216 via a zero-weight softmax net
    spec = {"input": [4], "layers": [CF.dense(4, 10), CF.softmax()], "lr": 0.1, "momentum": 0.0, "seed": 1}
    net = O.Net(spec)
    net.set(0, np.zeros(40, np.float32))
    loss = net.forward_backward(np.zeros((1, 4), np.float32), np.array([3], np.int32))
    assert rel_err(loss, np.log(10.0)) < 1e-6


def test_known_cd1_zero_fixed_point():  # test_energy.cpp:120-131
    recon, W, bv, bh, _ = O.rbm_cd1(np.zeros((2, 3), np.float32), np.zeros(3, np.float32), np.zeros(2, np.float32),
                                    np.full((4, 3), 0.5, np.float32), 0.1, O.canonical_f64(3, 8))
    assert not W.any() and not bv.any() and not bh.any()


def test_uniform_streams_match_reference_rng():
    """std::bernoulli_distribution == (generate_canonical<double,53> < p) over the same mt19937."""
    u = O.canonical_f64(5, 20000)
    bern = O.bernoulli_f32(5, 0.3, 10000)  # consumes one canonical double per draw
    assert np.array_equal(bern, (u[:10000] < 0.3).astype(np.float32))


@pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built (needs /root/reference)")
@pytest.mark.parametrize("name", ["mlp", "mnist_cnn", "cifar_cnn"])
def test_oracle_vs_live_reference(name):
    spec = CF.NET_CONFIGS[name](8)
    o, r = O.Net(spec), O.Net(spec, "ref")
    per = int(np.prod(spec["input"]))
    x = O.uniform_f32(7, 8 * per).reshape([8] + spec["input"])
    lab = O.uniform_int(8, 0, 9, 8)
    for _ in range(2):
        assert o.train_minibatch(x, lab) == r.train_minibatch(x, lab)
    for i in range(o.num_params()):
        assert bitwise(o.get(i), r.get(i))
