"""The oracle's Adagrad / Adadelta / Adam (optim.hpp:83-137) pinned bit-exactly to the reference:
golden fixtures (tests/golden/optim.npz from make_golden.py optim) and, where oracle/_ref is
built, the live reference."""
import json
from pathlib import Path

import numpy as np
import pytest

from oracle import oracle as O

GOLD = Path(__file__).resolve().parent / "golden"
META = json.loads((GOLD / "meta.json").read_text())


@pytest.mark.parametrize("kind", [1, 2, 3])
@pytest.mark.parametrize("name", ["mlp_small", "mnist_cnn_small"])
def test_optimizer_golden(kind, name):
    gold = np.load(GOLD / "optim.npz")
    g = np.load(GOLD / f"{name}.npz")
    net = O.Net(dict(META[name]["spec"], optimizer=kind, lr=0.01))
    losses = [net.train_minibatch(g["x"], g["labels"]) for _ in range(4)]
    assert np.array_equal(np.array(losses), gold[f"{name}_{kind}_losses"])
    for i in range(net.num_params()):
        for w in (0, 3, 4):
            assert np.array_equal(net.get(i, w).view(np.uint32), gold[f"{name}_{kind}_{w}_{i}"].view(np.uint32))


@pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built (needs /root/reference)")
@pytest.mark.parametrize("kind", [1, 2, 3])
def test_optimizer_vs_live_reference(kind):
    from paper_1804_04512_b200 import configs as CF
    spec = dict(CF.NET_CONFIGS["cifar_cnn"](8), optimizer=kind, lr=0.01)
    o, r = O.Net(spec), O.Net(spec, "ref")
    x = O.uniform_f32(7, 8 * 3072).reshape(8, 3, 32, 32)
    lab = O.uniform_int(8, 0, 9, 8)
    for _ in range(3):
        assert o.train_minibatch(x, lab) == r.train_minibatch(x, lab)
    for i in range(o.num_params()):
        for w in (0, 3, 4):
            assert np.array_equal(o.get(i, w).view(np.uint32), r.get(i, w).view(np.uint32)), (i, w)
