"""dbn_pretrain on the B200 (b2n_dbn_pretrain) vs the oracle's restatement, which is bit-exact to
the reference's own dbn_pretrain (tests/test_dbn.py). Same mt19937 uniform stream in the same
order; per-layer reconstruction errors within 1e-4 relative, trained parameters within the 1e-3
normalised bar (a Bernoulli draw within ~1e-7 of its probability could flip -- none do here)."""
import sys
from pathlib import Path

import numpy as np
import pytest

from conftest import norm_err
from oracle import oracle as O

pytestmark = pytest.mark.gpu
GOLD = Path(__file__).resolve().parent / "golden"
sys.path.insert(0, str(GOLD))
import make_golden as MG  # noqa: E402


def run_device(stack_np, data, epochs, lr, batch, seed):
    from paper_1804_04512_b200 import fastnn as F
    stack = []
    for W, bv, bh in stack_np:
        r = F.Rbm(W.shape[0], W.shape[1])
        r.set(W, bv, bh)
        stack.append(r)
    rep = F.dbn_pretrain(stack, data, epochs, lr, batch, F.Mt19937(seed))
    return [r.get() for r in stack], rep.recon


def compare(stack_np, data, epochs, lr, batch, seed):
    got, rg = run_device(stack_np, data, epochs, lr, batch, seed)
    want, rw = O.dbn_pretrain(stack_np, data, epochs, lr, batch, seed)
    for l in range(len(stack_np)):
        for e in range(epochs):
            assert abs(rg[l][e] - rw[l][e]) <= 1e-4 * abs(rw[l][e]), (l, e, rg[l][e], rw[l][e])
        for a, b in zip(got[l], want[l]):
            assert norm_err(a, b) < 1e-3, l


def test_dbn_golden_case(gpu):
    c = MG.DBN_CASE
    stack, data = MG.dbn_case_inputs()
    compare(stack, data, c["epochs"], c["lr"], c["batch"], c["seed"])
    g = np.load(GOLD / "dbn.npz")  # and against the reference's own numbers
    got, rg = run_device(stack, data, c["epochs"], c["lr"], c["batch"], c["seed"])
    assert np.allclose(np.array(rg), g["recon"], rtol=1e-4)


def test_dbn_mnist_shape(gpu):
    """the headline RBM shape as the first layer of a 784-500-250 stack, 1000 rows, batch 100"""
    dims = [784, 500, 250]
    stack = [(O.rbm_init(dims[l + 1], dims[l], 42 + l), np.zeros(dims[l], np.float32),
              np.zeros(dims[l + 1], np.float32)) for l in range(2)]
    data = O.bernoulli_f32(3, 0.3, 1000 * 784).reshape(1000, 784)
    compare(stack, data, 2, 0.1, 100, 5)


def test_dbn_errors(gpu):
    from paper_1804_04512_b200 import fastnn as F
    a, b = F.Rbm(24, 40), F.Rbm(16, 20)
    data = np.zeros((10, 40), np.float32)
    with pytest.raises(F.ShapeError, match="dbn_pretrain: layer 1 expects 20 visible units but layer 0 provides 24"):
        F.dbn_pretrain([a, b], data, 1, 0.1, 4, F.Mt19937(1))
    with pytest.raises(F.ParamError, match="empty stack"):
        F.dbn_pretrain([], data, 1, 0.1, 4, F.Mt19937(1))
    with pytest.raises(F.ParamError, match="batch_size"):
        F.dbn_pretrain([a], data, 1, 0.1, 0, F.Mt19937(1))
