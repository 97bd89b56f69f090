"""Convolutional RBM (crbm_cd_update, energy.hpp:333-376): the oracle restatement
(oracle/fastnn_oracle.cpp orc_crbm_cd1) pinned bit-exact to the reference's golden fixtures
(tests/golden/crbm.npz, made by tests/golden/make_golden.py crbm from the unmodified reference),
to the reference's own known-answer tests (test_energy.cpp:347-503) and, where oracle/_ref is
built, to the reference live on random shapes."""
import sys
from pathlib import Path

import numpy as np
import pytest

from conftest import rel_err
from oracle import oracle as O

GOLD = Path(__file__).resolve().parent / "golden"
sys.path.insert(0, str(GOLD))
from make_golden import CRBM_CASES  # noqa: E402


def bitwise(a, b):
    a, b = np.asarray(a), np.asarray(b)
    return a.shape == b.shape and np.array_equal(a.view(np.uint32), b.view(np.uint32))


@pytest.mark.parametrize("i", range(len(CRBM_CASES)))
def test_crbm_golden(i):
    """the reference consumes its std::mt19937(5 + i); the oracle takes the same
    generate_canonical<double,53> stream as supplied uniforms and matches bit for bit"""
    g = np.load(GOLD / "crbm.npz")
    c, h, w, k, kh, kw, B = CRBM_CASES[i]
    u = O.canonical_f64(5 + i, B * k * (h - kh + 1) * (w - kw + 1))
    recon, k1, bv1, bh1, _ = O.crbm_cd1(g[f"ker{i}"], g[f"bv{i}"], g[f"bh{i}"], g[f"v0_{i}"], 0.1, u)
    assert bitwise(k1, g[f"ker1_{i}"]) and bitwise(bv1, g[f"bv1_{i}"]) and bitwise(bh1, g[f"bh1_{i}"])
    assert recon == g[f"recon{i}"][0]


def test_crbm_init_matches_reference_glorot():
    g = np.load(GOLD / "crbm.npz")
    for i, (c, h, w, k, kh, kw, _) in enumerate(CRBM_CASES):
        assert bitwise(O.crbm_init(c, h, w, k, kh, kw, 42 + i), g[f"ker{i}"])


def test_zero_model_hidden_means_one_half():  # test_energy.cpp:348-363
    ker = np.zeros((2, 1, 3, 3), np.float32)
    v0 = O.uniform_f32(19, 2 * 25).reshape(2, 1, 5, 5)
    u = O.canonical_f64(1, 2 * 2 * 9)
    _, _, _, _, ex = O.crbm_cd1(ker, np.zeros(1, np.float32), np.zeros(2, np.float32), v0, 0.1, u)
    assert np.all(ex["h0"] == 0.5)


def test_one_by_one_degenerates_to_dense_rbm():  # test_energy.cpp:466-503 / acceptance criterion 7
    H, V, B = 2, 3, 4
    W = O.rbm_init(H, V, 23)
    v = O.bernoulli_f32(24, 0.5, B * V).reshape(B, V)
    u = O.canonical_f64(25, B * H)
    rd, Wd, bvd, bhd, _ = O.rbm_cd1(W, np.zeros(V, np.float32), np.zeros(H, np.float32), v, 0.1, u.reshape(B, H))
    rc, kc, bvc, bhc, _ = O.crbm_cd1(W.reshape(H, V, 1, 1), np.zeros(V, np.float32), np.zeros(H, np.float32),
                                     v.reshape(B, V, 1, 1), 0.1, u)
    assert abs(rd - rc) < 1e-9
    assert np.abs(Wd - kc.reshape(H, V)).max() < 1e-6
    assert np.abs(bvd - bvc).max() < 1e-6 and np.abs(bhd - bhc).max() < 1e-6


def test_toy_training_reduces_reconstruction():  # test_energy.cpp:437-464
    c, h, w, k, kh, kw, B = 1, 6, 6, 4, 3, 3, 8
    ker = O.crbm_init(c, h, w, k, kh, kw, 22)
    bv, bh = np.zeros(c, np.float32), np.zeros(k, np.float32)
    data = O.bernoulli_f32(23, 0.4, B * h * w).reshape(B, c, h, w)
    errs = []
    for epoch in range(50):
        u = O.canonical_f64(100 + epoch, B * k * 16)
        r, ker, bv, bh, _ = O.crbm_cd1(ker, bv, bh, data, 0.05, u)
        errs.append(r)
    assert errs[-1] < errs[0]


def test_shard_deltas_sum_to_the_full_batch_update():
    """data-parallel form: per-shard deltas (lr / B_global) summed over shards == the full-batch
    update within fp32 reassociation"""
    c, h, w, k, kh, kw, B = 2, 8, 7, 3, 3, 2, 6
    ker = O.crbm_init(c, h, w, k, kh, kw, 5)
    bv = O.uniform_f32(1, c, -0.1, 0.1)
    bh = O.uniform_f32(2, k, -0.1, 0.1)
    v0 = O.bernoulli_f32(3, 0.5, B * c * h * w).reshape(B, c, h, w)
    per = k * (h - kh + 1) * (w - kw + 1)
    u = O.canonical_f64(4, B * per)
    r, k1, bv1, bh1, _ = O.crbm_cd1(ker, bv, bh, v0, 0.1, u)
    dk, dbv, dbh, rs = 0, 0, 0, 0.0
    for lo in (0, 3):
        rr, _, _, _, ex = O.crbm_cd1(ker, bv, bh, v0[lo:lo + 3], 0.1, u[lo * per:(lo + 3) * per], b_global=B,
                                     deltas=True)
        dk, dbv, dbh, rs = dk + ex["dker"], dbv + ex["dbv"], dbh + ex["dbh"], rs + rr
    assert np.abs(ker + dk - k1).max() < 1e-6 and np.abs(bv + dbv - bv1).max() < 1e-6
    assert np.abs(bh + dbh - bh1).max() < 1e-6 and abs(rs - r) < 1e-9


@pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built (needs /root/reference)")
@pytest.mark.parametrize("shape", [(2, 9, 7, 5, 3, 3, 3), (3, 11, 10, 4, 2, 3, 2), (1, 16, 16, 8, 5, 5, 2)])
def test_oracle_vs_live_reference(shape):
    c, h, w, k, kh, kw, B = shape
    ker = O.crbm_init(c, h, w, k, kh, kw, 42, "ref")
    bv = O.uniform_f32(7, c, -0.1, 0.1)
    bh = O.uniform_f32(8, k, -0.1, 0.1)
    v0 = O.bernoulli_f32(3, 0.5, B * c * h * w).reshape(B, c, h, w)
    u = O.canonical_f64(5, B * k * (h - kh + 1) * (w - kw + 1))
    r1, k1, bv1, bh1, _ = O.crbm_cd1(ker, bv, bh, v0, 0.1, u)
    r2, k2, bv2, bh2 = O.ref_crbm_cd(ker, bv, bh, v0, 0.1, 5)
    # bit-exact on the kernels / bv / recon; the reference's direct-conv backend may round the
    # hidden means of multi-channel odd-width maps differently by one ulp, seen in bh only
    assert bitwise(k1, k2) and bitwise(bv1, bv2) and r1 == r2
    assert rel_err(bh1, bh2) < 1e-6
