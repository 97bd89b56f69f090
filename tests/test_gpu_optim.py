"""Adagrad / Adadelta / Adam (optim.hpp:83-137) on the B200: the step runs SPLIT (backward writes the
packed gradient) + one packed optimizer kernel; parameters and optimizer state vs the oracle, which
is bit-exact to the reference for all three (tests/test_optim.py). Tolerance: the 1e-3 normalised bar
(3xTF32 gradients feed the elementwise updates)."""
import json
from pathlib import Path

import numpy as np
import pytest

from conftest import norm_err
from oracle import oracle as O
from paper_1804_04512_b200 import configs as CF

pytestmark = pytest.mark.gpu
GOLD = Path(__file__).resolve().parent / "golden"
META = json.loads((GOLD / "meta.json").read_text())
KINDS = {"adagrad": 1, "adadelta": 2, "adam": 3}


def pair(spec):
    from paper_1804_04512_b200 import fastnn as F
    net = F.build_network(spec)
    orc = O.Net(spec)
    for i in range(net.num_params()):
        net.set_param(i, orc.get(i))
    return net, orc


@pytest.mark.parametrize("kind", list(KINDS))
@pytest.mark.parametrize("name", ["mlp_small", "mnist_cnn_small", "cifar_cnn_small", "imagenet_cnn_small"])
def test_optimizer_steps(gpu, kind, name):
    from paper_1804_04512_b200 import fastnn as F
    spec = dict(META[name]["spec"], optimizer=KINDS[kind], lr=0.01)
    g = np.load(GOLD / f"{name}.npz")
    net, orc = pair(spec)
    for step in range(4):
        lg = F.train_minibatch_labels(net, g["x"], g["labels"])
        lo = orc.train_minibatch(g["x"], g["labels"])
        assert abs(lg - lo) / lo < 1e-4, (step, lg, lo)
    for i in range(net.num_params()):
        assert norm_err(net.get_param(i).ravel(), orc.get(i)) < 1e-3, i
        assert norm_err(net.get_param(i, F.OPT_STATE1).ravel(), orc.get(i, 3)) < 1e-3, i
        if kind != "adagrad":
            assert norm_err(net.get_param(i, F.OPT_STATE2).ravel(), orc.get(i, 4)) < 1e-3, i


@pytest.mark.parametrize("kind", list(KINDS))
def test_optimizer_full_mlp_staged(gpu, kind):
    """config-1 shapes, device-resident stepping (graph replays advance adam's step counter)"""
    from paper_1804_04512_b200 import fastnn as F
    spec = dict(CF.NET_CONFIGS["mlp"](100), optimizer=KINDS[kind], lr=0.001)
    x = O.uniform_f32(1, 100 * 784).reshape(100, 784)
    lab = O.uniform_int(2, 0, 9, 100)
    net, orc = pair(spec)
    net.stage(x, lab)
    net.run_staged(5)
    for _ in range(5):
        lo = orc.train_minibatch(x, lab)
    assert abs(net.loss() - lo) / lo < 1e-4
    for i in range(net.num_params()):
        assert norm_err(net.get_param(i).ravel(), orc.get(i)) < 1e-3, i


def test_adam_fit_and_resume(gpu, tmp_path):
    """fit with adam vs the oracle; then save with state, reload into a fresh net, and one more
    epoch on both lands on identical parameters"""
    from paper_1804_04512_b200 import fastnn as F
    spec = dict(META["mnist_cnn_small"]["spec"], optimizer=3, lr=0.01, batch_size=16)
    N = 70
    x = O.uniform_f32(31, N * 144).reshape(N, 1, 12, 12)
    lab = O.uniform_int(32, 0, 9, N)
    net, orc = pair(spec)
    rep = F.fit(net, x, lab, 2)
    loss, acc = orc.fit(x, lab, 16, spec["seed"], 2)
    for e in range(2):
        assert abs(rep.epochs[e].loss - loss[e]) / loss[e] < 1e-4
    for i in range(net.num_params()):
        assert norm_err(net.get_param(i).ravel(), orc.get(i)) < 1e-3, i
    F.save_network(net, tmp_path / "a.fnn1", with_state=True)
    other = F.build_network(spec)
    F.load_network(other, tmp_path / "a.fnn1", with_state=True)
    la = [F.train_minibatch_labels(net, x[:16], lab[:16]) for _ in range(3)]
    lb = [F.train_minibatch_labels(other, x[:16], lab[:16]) for _ in range(3)]
    assert la == lb
    for i in range(net.num_params()):
        assert np.array_equal(net.get_param(i), other.get_param(i))
        assert np.array_equal(net.get_param(i, F.OPT_STATE2), other.get_param(i, F.OPT_STATE2))


def test_optimizer_views_and_errors(gpu):
    from paper_1804_04512_b200 import fastnn as F
    net = F.build_network(dict(META["mlp_small"]["spec"]))
    with pytest.raises(F.BoundsError):
        net.get_param(0, F.OPT_STATE1)  # SGD has no adagrad/adam state
    with pytest.raises(F.SpecError):
        F.build_network(dict(META["mlp_small"]["spec"], optimizer=7))
    bad = F.build_network(dict(META["mlp_small"]["spec"], optimizer=3, lr=-1.0))
    with pytest.raises(F.ParamError):  # optim.hpp:51-55
        F.train_minibatch_labels(bad, np.zeros((2, 64), np.float32), np.zeros(2, np.int32))
