"""Convolutional RBM CD-1 on the B200 (crbm.cuh: tcgen05 implicit-GEMM conv kernels) vs the oracle
restatement of crbm_cd_update (energy.hpp:333-376). Sampling contract: hs == (u < h0) bit-exactly
on the kernel's own h0; where the kernel's h0 and the oracle's straddle a uniform (a flip inside the
probability error band), the oracle is re-run on the kernel's sample so the rest of the step is
still compared. Tolerances: chain means 1e-5, parameter deltas 1e-3 (north_star's 1e-3 bar; the
convs run 3xTF32), recon 1e-5 relative."""
import sys
from pathlib import Path

import numpy as np
import pytest

from conftest import norm_err
from oracle import oracle as O

sys.path.insert(0, str(Path(__file__).resolve().parent / "golden"))
from make_golden import CRBM_CASES  # noqa: E402

pytestmark = pytest.mark.gpu

SHAPES = CRBM_CASES + [(1, 28, 28, 12, 5, 5, 100), (3, 32, 32, 8, 5, 5, 16), (16, 12, 12, 16, 3, 3, 10),
                       (1, 28, 28, 32, 3, 3, 7), (2, 5, 40, 3, 1, 7, 5),
                       # more images than co-resident CTAs (a CTA loops over images; the last CTA's
                       # partial rows no longer fit its shared memory: the global-load reduction)
                       (1, 28, 28, 12, 5, 5, 400),
                       # widest register strip template (kw = 8) and a 1-wide kernel on a tall map
                       (2, 20, 23, 4, 3, 8, 6), (1, 30, 9, 5, 4, 1, 3)]


def _step(c, h, w, k, kh, kw, B, lr=0.1, seed=0):
    from paper_1804_04512_b200 import fastnn as F
    m = F.Crbm(c, h, w, k, kh, kw)
    m.keep_states(True)
    ker = O.crbm_init(c, h, w, k, kh, kw, 42 + seed)
    bv = O.uniform_f32(7 + seed, c, -0.1, 0.1)
    bh = O.uniform_f32(8 + seed, k, -0.1, 0.1)
    m.set(ker, bv, bh)
    v0 = O.bernoulli_f32(3 + seed, 0.5, B * c * h * w).reshape(B, c, h, w)
    u = O.canonical_f64(5 + seed, B * k * (h - kh + 1) * (w - kw + 1))
    recon = F.crbm_cd_update(m, v0, lr, u)
    return m, (ker, bv, bh), v0, u, recon


@pytest.fixture(params=["fused", "split"])
def crbm_path(request, monkeypatch):
    """the one-launch per-image step (crbm_fused.cuh) and the tensor-core split path (crbm.cuh)"""
    if request.param == "split":
        monkeypatch.setenv("B2N_CRBM_FUSED", "0")
    return request.param


@pytest.mark.parametrize("shape", SHAPES)
def test_crbm_cd1_step(gpu, shape, crbm_path):
    c, h, w, k, kh, kw, B = shape
    m, (ker, bv, bh), v0, u, recon_g = _step(*shape)
    h0, hs, v1, h1 = m.last_states(B)
    uu = u.reshape(h0.shape)
    np.testing.assert_array_equal(hs, (uu < h0.astype(np.float64)).astype(np.float32))
    _, _, _, _, ex = O.crbm_cd1(ker, bv, bh, v0, 0.1, u)
    assert norm_err(h0, ex["h0"]) < 1e-5
    flips = hs != ex["hs"]
    dp = np.abs(h0 - ex["h0"]).max()
    assert np.all(np.abs(uu[flips] - ex["h0"][flips]) <= dp + 1e-7), "flip outside the probability error band"
    # the oracle on the kernel's own sample (u forced to 0 / 2 on the flipped units)
    u2 = np.where(flips, np.where(hs > 0, 0.0, 2.0), uu).ravel()
    recon_o, ko, bvo, bho, ex = O.crbm_cd1(ker, bv, bh, v0, 0.1, u2)
    np.testing.assert_array_equal(hs, ex["hs"])
    assert norm_err(v1, ex["v1"]) < 1e-5
    assert norm_err(h1, ex["h1"]) < 1e-5
    kg, bvg, bhg = m.get()
    assert norm_err(kg - ker, ko - ker) < 1e-3
    assert norm_err(bvg - bv, bvo - bv) < 1e-3
    assert norm_err(bhg - bh, bho - bh) < 1e-3
    assert abs(recon_g - recon_o) <= 1e-5 * max(recon_o, 1e-12)


def test_crbm_init_matches_oracle(gpu):
    from paper_1804_04512_b200 import fastnn as F
    m = F.Crbm(3, 32, 32, 8, 5, 5)
    m.init(42)
    ker, bv, bh = m.get()
    np.testing.assert_array_equal(ker, O.crbm_init(3, 32, 32, 8, 5, 5, 42))
    assert not bv.any() and not bh.any()


def test_crbm_zero_model_hidden_means_one_half(gpu):  # test_energy.cpp:348-363
    from paper_1804_04512_b200 import fastnn as F
    m = F.Crbm(1, 5, 5, 2, 3, 3)
    m.keep_states(True)
    m.set(np.zeros((2, 1, 3, 3), np.float32), np.zeros(1, np.float32), np.zeros(2, np.float32))
    v0 = O.uniform_f32(19, 50).reshape(2, 1, 5, 5)
    F.crbm_cd_update(m, v0, 0.1, O.canonical_f64(1, 2 * 2 * 9))
    h0, _, _, _ = m.last_states(2)
    assert np.all(h0 == 0.5)


def test_crbm_one_by_one_matches_dense_rbm(gpu, crbm_path):  # test_energy.cpp:466-503
    from paper_1804_04512_b200 import fastnn as F
    H, V, B = 2, 3, 4
    W = O.rbm_init(H, V, 23)
    v = O.bernoulli_f32(24, 0.5, B * V).reshape(B, V)
    u = O.canonical_f64(25, B * H)
    d = F.Rbm(H, V)
    d.set(W, np.zeros(V, np.float32), np.zeros(H, np.float32))
    c = F.Crbm(V, 1, 1, H, 1, 1)
    c.set(W.reshape(H, V, 1, 1), np.zeros(V, np.float32), np.zeros(H, np.float32))
    rd = F.cd_k_update(d, v, 1, 0.1, u.reshape(B, H))
    rc = F.crbm_cd_update(c, v.reshape(B, V, 1, 1), 0.1, u)
    assert abs(rd - rc) < 1e-6
    wd, bvd, bhd = d.get()
    kc, bvc, bhc = c.get()
    assert np.abs(wd - kc.reshape(H, V)).max() < 1e-6
    assert np.abs(bvd - bvc).max() < 1e-6 and np.abs(bhd - bhc).max() < 1e-6


def test_crbm_training_reduces_reconstruction(gpu):  # test_energy.cpp:437-464
    from paper_1804_04512_b200 import fastnn as F
    m = F.Crbm(1, 6, 6, 4, 3, 3)
    m.init(22)
    data = O.bernoulli_f32(23, 0.4, 8 * 36).reshape(8, 1, 6, 6)
    errs = [F.crbm_cd_update(m, data, 0.05, O.canonical_f64(100 + e, 8 * 4 * 16)) for e in range(50)]
    assert errs[-1] < errs[0]


def test_crbm_staged_steps_match_calls(gpu, crbm_path):
    """run_staged(n) replays the captured step graph: same arithmetic as n cd_update calls"""
    from paper_1804_04512_b200 import fastnn as F
    c, h, w, k, kh, kw, B = 1, 28, 28, 12, 5, 5, 100
    v0 = O.bernoulli_f32(3, 0.5, B * c * h * w).reshape(B, c, h, w)
    u = O.canonical_f64(5, B * k * 24 * 24)
    a, b = F.Crbm(c, h, w, k, kh, kw), F.Crbm(c, h, w, k, kh, kw)
    a.init(42)
    b.init(42)
    for _ in range(3):
        ra = F.crbm_cd_update(a, v0, 0.1, u)
    b.stage(v0, u)
    b.run_staged(3, 0.1)
    assert b.recon() == ra
    for x, y in zip(a.get(), b.get()):
        np.testing.assert_array_equal(x, y)


def test_crbm_fused_is_one_launch_and_matches_split(gpu):
    """the MNIST-shape CRBM takes the one-launch path; it agrees with the split tensor-core path"""
    import os
    from paper_1804_04512_b200 import fastnn as F
    c, h, w, k, kh, kw, B = 1, 28, 28, 12, 5, 5, 100
    v0 = O.bernoulli_f32(3, 0.5, B * c * h * w).reshape(B, c, h, w)
    u = O.canonical_f64(5, B * k * 24 * 24)
    a = F.Crbm(c, h, w, k, kh, kw)
    a.init(42)
    ra = F.crbm_cd_update(a, v0, 0.1, u)
    assert a.kernels_per_step() == 1
    os.environ["B2N_CRBM_FUSED"] = "0"
    try:
        b = F.Crbm(c, h, w, k, kh, kw)
        b.init(42)
        rb = F.crbm_cd_update(b, v0, 0.1, u)
        assert b.kernels_per_step() == 5
    finally:
        del os.environ["B2N_CRBM_FUSED"]
    ka, kb = a.get()[0], b.get()[0]
    k0 = O.crbm_init(c, h, w, k, kh, kw, 42)
    assert norm_err(ka - k0, kb - k0) < 1e-3
    assert abs(ra - rb) <= 1e-5 * rb


def test_crbm_last_states_needs_keep(gpu):
    from paper_1804_04512_b200 import fastnn as F
    m = F.Crbm(1, 6, 6, 2, 3, 3)
    F.crbm_cd_update(m, np.zeros((2, 1, 6, 6), np.float32), 0.1, np.zeros(2 * 2 * 16))
    with pytest.raises(F.ParamError):
        m.last_states(2)


def test_crbm_shape_errors(gpu):
    from paper_1804_04512_b200 import fastnn as F
    with pytest.raises(F.ShapeError, match="kernel extents exceed visible extents"):
        F.Crbm(1, 4, 4, 1, 5, 5)
    with pytest.raises(F.ShapeError):
        F.Crbm(1, 28, 28, 40, 9, 9)  # k*kh*kw beyond the tensor-core conv envelope: loud, no fallback
    m = F.Crbm(1, 6, 6, 2, 3, 3)
    with pytest.raises(F.ShapeError):
        F.crbm_cd_update(m, np.zeros((2, 1, 5, 6), np.float32), 0.1, np.zeros(64))
