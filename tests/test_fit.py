"""fit / evaluate / BatchIterator (network.hpp:474-511, data.hpp:224-266): the oracle's restatement
pinned to the reference's own fit on golden fixtures (tests/golden/fit.npz, make_golden.py fit), and
the library's host-side batch order (b2n_batch_order, no GPU needed) equal to BatchIterator's."""
import json
from pathlib import Path

import numpy as np
import pytest

from oracle import oracle as O

GOLD = Path(__file__).resolve().parent / "golden"
META = json.loads((GOLD / "meta.json").read_text())
FIT_CASES = {"mlp_small": (250, 32, 3), "mnist_cnn_small": (90, 20, 2)}  # make_golden.FIT_CASES
ORDERS = [(250, 42), (90, 7), (1000, 3)]


@pytest.mark.parametrize("n,seed", ORDERS)
def test_oracle_batch_order_golden(n, seed):
    g = np.load(GOLD / "fit.npz")
    for e in range(3):
        assert np.array_equal(O.batch_order(n, seed, e), g[f"order_{n}_{seed}_{e}"])


@pytest.mark.parametrize("n,seed", ORDERS)
def test_library_batch_order_golden(n, seed):
    from paper_1804_04512_b200 import fastnn as F
    g = np.load(GOLD / "fit.npz")
    for e in range(3):
        assert np.array_equal(F.batch_order(n, seed, e), g[f"order_{n}_{seed}_{e}"])


@pytest.mark.parametrize("name", list(FIT_CASES))
def test_oracle_fit_golden(name):
    g = np.load(GOLD / "fit.npz")
    N, B, epochs = FIT_CASES[name]
    spec = META[name]["spec"]
    net = O.Net(spec)
    x, lab = g[f"{name}_x"], g[f"{name}_labels"]
    assert net.evaluate(x, lab, B) == g[f"{name}_acc0"][0]
    loss, acc = net.fit(x, lab, B, spec["seed"], epochs)
    assert np.array_equal(loss, g[f"{name}_loss"])  # bit-exact, as every oracle step is
    assert np.array_equal(acc, g[f"{name}_acc"])
    for i in range(net.num_params()):
        assert np.array_equal(net.get(i).view(np.uint32), g[f"{name}_final{i}"].view(np.uint32)), i


@pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built (needs /root/reference)")
def test_oracle_fit_vs_live_reference():
    from paper_1804_04512_b200 import configs as CF
    spec = CF.NET_CONFIGS["mlp"](50)
    o, r = O.Net(spec), O.Net(spec, "ref")
    N = 130
    x = O.uniform_f32(5, N * 784).reshape(N, 784)
    lab = O.uniform_int(6, 0, 9, N)
    lo, ao = o.fit(x, lab, 50, 42, 2)
    lr_, ar = r.fit(x, lab, 50, 42, 2)
    assert np.array_equal(lo, lr_) and np.array_equal(ao, ar)
