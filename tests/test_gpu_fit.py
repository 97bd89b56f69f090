"""Device-resident fit / evaluate (b2n_net_fit / b2n_net_evaluate) vs the oracle's fit, which is
pinned bit-exactly to the reference's fastnn::fit (tests/test_fit.py). Same shuffled batch order,
same partial last batch, per-epoch loss within 1e-4 relative, train accuracy within one sample
(an argmax near-tie may flip under 3xTF32), parameters within the 1e-3 normalised bar."""
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


def run_pair(spec, B, x, lab, epochs):
    from paper_1804_04512_b200 import fastnn as F
    spec = dict(spec, batch_size=B)
    net = F.build_network(spec)
    orc = O.Net(spec)
    for i in range(net.num_params()):
        net.set_param(i, orc.get(i).reshape(net.param_shape(i)))
    rep = F.fit(net, x, lab, epochs)
    loss, acc = orc.fit(x, lab, B, spec.get("seed", 42), epochs)
    N = lab.shape[0]
    for e in range(epochs):
        st = rep.epochs[e]
        assert abs(st.loss - loss[e]) / loss[e] < 1e-4, (e, st.loss, loss[e])
        assert abs(st.accuracy - acc[e]) <= 1.0 / N + 1e-12, (e, st.accuracy, acc[e])
        assert st.seconds > 0
    assert rep.total_batches == epochs * -(-N // B)
    for i in range(net.num_params()):
        e = norm_err(net.get_param(i).ravel(), orc.get(i))
        assert e < 1e-3, (i, e)
    return net, orc


@pytest.mark.parametrize("name,N,B,epochs", [("mlp_small", 250, 32, 3), ("mnist_cnn_small", 90, 20, 2),
                                             ("cifar_cnn_small", 70, 16, 2), ("imagenet_cnn_small", 40, 12, 2)])
def test_fit_small(gpu, name, N, B, epochs):
    spec = META[name]["spec"]
    per = int(np.prod(spec["input"]))
    x = O.uniform_f32(201, N * per).reshape([N] + spec["input"])
    lab = O.uniform_int(202, 0, 9, N)
    run_pair(spec, B, x, lab, epochs)


@pytest.mark.parametrize("name", ["mlp", "mnist_cnn"])
def test_fit_full_config(gpu, name):
    """the configs' real shapes (batch 100) on 550 samples: five full batches and a partial one"""
    spec = CF.NET_CONFIGS[name](100)
    N = 550
    per = int(np.prod(spec["input"]))
    x = O.uniform_f32(11, N * per).reshape([N] + spec["input"])
    lab = O.uniform_int(12, 0, 9, N)
    run_pair(spec, 100, x, lab, 2)


def test_evaluate_and_refit(gpu):
    """evaluate in dataset order; a second, larger dataset reallocates the resident copy"""
    from paper_1804_04512_b200 import fastnn as F
    spec = dict(META["mlp_small"]["spec"], batch_size=32)
    net = F.build_network(spec)
    orc = O.Net(spec)
    for n in (70, 300, 33):
        x = O.uniform_f32(n, n * 64).reshape(n, 64)
        lab = O.uniform_int(n + 1, 0, 9, n)
        assert F.evaluate(net, x, lab) == orc.evaluate(x, lab, 32)
        F.fit(net, x, lab, 1)
        orc.fit(x, lab, 32, 42, 1)
        for i in range(net.num_params()):
            assert norm_err(net.get_param(i).ravel(), orc.get(i)) < 1e-3


def test_fit_errors(gpu):
    from paper_1804_04512_b200 import fastnn as F
    net = F.build_network(dict(META["mlp_small"]["spec"], batch_size=8))
    x = np.zeros((10, 64), np.float32)
    with pytest.raises(F.ConsistencyError):  # data.hpp:257-260
        F.fit(net, x, np.full(10, 10, np.int32), 1)
    with pytest.raises(F.ParamError):
        F.fit(net, x, np.zeros(10, np.int32), 0)
    with pytest.raises(F.DataError):
        F.evaluate(net, x[:0], np.zeros(0, np.int32))
