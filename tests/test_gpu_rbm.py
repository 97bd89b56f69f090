"""RBM CD-1 (config 2) on the B200 vs the oracle restatement of cd_k_update (energy.hpp:131-171).
Sampling contract: hs == (u < h0) bit-exactly on the kernel's own h0; cross-implementation flips
only where |u - p_ref| is within the probability error."""
import numpy as np
import pytest

from conftest import norm_err
from oracle import oracle as O

pytestmark = pytest.mark.gpu


def check_rbm_step(rbm, W, bv, bh, v0, u, k, recon_g, hs_levels):
    """Asserts every output of one GPU CD-k step against the oracle re-run on the kernel's OWN
    samples (hs_levels[s] = the kernel's hidden sample of Gibbs step s): sampling decisions are
    checked separately, so the W / bias / v1 / recon comparison never depends on a flip-free draw."""
    B, H = v0.shape[0], W.shape[0]
    u = np.asarray(u, np.float64).reshape(k, B, H)
    _, _, _, _, ex = O.rbm_cdk(W, bv, bh, v0, k, 0.1, u)
    # flips vs the oracle's own samples are confined to the probability error band (last level)
    h0_g = rbm.last_states(B)[0]
    assert norm_err(h0_g, ex["h0"]) < 1e-5
    flips = hs_levels[-1] != ex["hs"]
    nflip = int(flips.sum())
    if k == 1:
        dp = np.abs(h0_g - ex["h0"]).max()
        assert np.all(np.abs(u[0][flips] - ex["h0"][flips]) <= dp + 1e-7), "flip outside the probability error band"
    assert nflip <= max(2, B * H // 1000), nflip
    uf = np.stack([O.force_samples(u[s], hs_levels[s]) for s in range(k)])
    recon_o, Wo, bvo, bho, ex2 = O.rbm_cdk(W, bv, bh, v0, k, 0.1, uf)
    np.testing.assert_array_equal(ex2["hs"], hs_levels[-1])
    _, _, v1_g, h1_g = rbm.last_states(B)
    assert norm_err(v1_g, ex2["v1"] if k == 1 else ex2["vk"]) < 1e-4  # the last visible means
    assert norm_err(h1_g, ex2["h1"]) < 1e-4
    wg, bvg, bhg = rbm.get()
    assert norm_err(wg - W, Wo - W) < 1e-3
    assert norm_err(bvg - bv, bvo - bv) < 1e-3
    assert norm_err(bhg - bh, bho - bh) < 1e-3
    assert norm_err(wg, Wo) < 1e-5
    assert abs(recon_g - recon_o) / recon_o < 1e-5
    return nflip


@pytest.mark.parametrize("B,H,V", [(100, 500, 784), (10, 50, 78), (1, 8, 4), (130, 64, 100)])
def test_cd1_step(gpu, B, H, V):
    from paper_1804_04512_b200 import fastnn as F
    rbm = F.Rbm(H, V)
    rbm.init(42)
    W = O.rbm_init(H, V, 42)
    w0, bv0, bh0 = rbm.get()
    np.testing.assert_array_equal(w0, W)
    v0 = O.bernoulli_f32(3, 0.5, B * V).reshape(B, V)
    u = O.canonical_f64(5, B * H).reshape(B, H)
    bv = np.zeros(V, np.float32)
    bh = np.zeros(H, np.float32)
    recon_g = F.cd_k_update(rbm, v0, 1, 0.1, u)
    h0, hs, v1, h1 = rbm.last_states(B)
    # bit-exact sampling on the kernel's own probabilities
    np.testing.assert_array_equal(hs, (u < h0.astype(np.float64)).astype(np.float32))
    nflip = check_rbm_step(rbm, W, bv, bh, v0, u, 1, recon_g, [hs])
    print(f"B={B} H={H} V={V}: {nflip} sample flips vs the oracle's probabilities (re-run on the kernel's samples)")


@pytest.mark.parametrize("fused", ["1", "0"])
def test_cd1_step_nonzero_biases_three_steps(gpu, fused, monkeypatch):
    """three consecutive full-size CD-1 steps from non-zero biases (fused and split paths), every
    step asserted against the oracle continued from the GPU's own parameters"""
    from paper_1804_04512_b200 import fastnn as F
    monkeypatch.setenv("B2N_RBM_FUSED", fused)
    B, H, V = 100, 500, 784
    rbm = F.Rbm(H, V)
    W = O.rbm_init(H, V, 42)
    bv = O.uniform_f32(7, V, -0.5, 0.5)
    bh = O.uniform_f32(8, H, -0.5, 0.5)
    rbm.set(W, bv, bh)
    for step in range(3):
        W, bv, bh = rbm.get()
        v0 = O.bernoulli_f32(20 + step, 0.3, B * V).reshape(B, V)
        u = O.canonical_f64(30 + step, B * H).reshape(B, H)
        recon_g = F.cd_k_update(rbm, v0, 1, 0.1, u)
        h0, hs, _, _ = rbm.last_states(B)
        np.testing.assert_array_equal(hs, (u < h0.astype(np.float64)).astype(np.float32))
        check_rbm_step(rbm, W, bv, bh, v0, u, 1, recon_g, [hs])


@pytest.mark.parametrize("B,H,V", [(100, 500, 784), (20, 64, 100)])
def test_cdk2_step(gpu, B, H, V, monkeypatch):
    """CD-k with k = 2 (energy.hpp:139-144): the chain resamples hs from v1 with the second block
    of k * B * H uniforms. The first-level samples are read from a k = 1 step on an identical
    model (same split-path GEMM, deterministic), the second from the k = 2 step itself."""
    from paper_1804_04512_b200 import fastnn as F
    monkeypatch.setenv("B2N_RBM_FUSED", "0")
    W = O.rbm_init(H, V, 42)
    bv = O.uniform_f32(7, V, -0.2, 0.2)
    bh = O.uniform_f32(8, H, -0.2, 0.2)
    v0 = O.bernoulli_f32(3, 0.5, B * V).reshape(B, V)
    u = O.canonical_f64(5, 2 * B * H).reshape(2, B, H)
    a, b = F.Rbm(H, V), F.Rbm(H, V)
    a.set(W, bv, bh)
    b.set(W, bv, bh)
    F.cd_k_update(a, v0, 1, 0.1, u[0])
    h0a, hs1, _, _ = a.last_states(B)
    np.testing.assert_array_equal(hs1, (u[0] < h0a.astype(np.float64)).astype(np.float32))
    recon_g = F.cd_k_update(b, v0, 2, 0.1, u)
    h0b, hs2, _, _ = b.last_states(B)
    np.testing.assert_array_equal(h0a, h0b)
    nflip = check_rbm_step(b, W, bv, bh, v0, u, 2, recon_g, [hs1, hs2])
    print(f"CD-2 B={B}: {nflip} last-level flips vs the oracle's own chain")


def test_cd1_zero_model_fixed_point(gpu):
    """test_energy.cpp:120-131: v0 = 0.5 on the zero model gives a zero update."""
    from paper_1804_04512_b200 import fastnn as F
    rbm = F.Rbm(2, 3)
    rbm.set(np.zeros((2, 3), np.float32), np.zeros(3, np.float32), np.zeros(2, np.float32))
    v0 = np.full((4, 3), 0.5, np.float32)
    u = O.canonical_f64(3, 8)
    F.cd_k_update(rbm, v0, 1, 0.1, u)
    w, bv, bh = rbm.get()
    assert not w.any() and not bv.any() and not bh.any()


def test_k_below_one(gpu):
    from paper_1804_04512_b200 import fastnn as F
    rbm = F.Rbm(2, 2)
    with pytest.raises(F.ParamError):
        F.cd_k_update(rbm, np.zeros((1, 2), np.float32), 0, 0.1, np.zeros(2))


def test_zero_copy_pinned_inputs_match_staged(gpu):
    """pinned caller buffers take the zero-copy fused launch (the kernel reads v0 and the uniforms
    from host memory); pageable ones are staged by copies. Same kernel arithmetic: bitwise equal."""
    import torch
    from paper_1804_04512_b200 import fastnn as F
    B, V, H = 100, 784, 500
    v0 = O.bernoulli_f32(3, 0.5, B * V).reshape(B, V)
    u = O.canonical_f64(5, B * H).reshape(B, H)
    v0p = torch.empty((B, V), dtype=torch.float32, pin_memory=True).numpy()
    up = torch.empty((B, H), dtype=torch.float64, pin_memory=True).numpy()
    v0p[:] = v0
    up[:] = u
    a, b = F.Rbm(H, V), F.Rbm(H, V)
    a.init(42)
    b.init(42)
    for step in range(3):
        ra = F.cd_k_update(a, v0, 1, 0.1, u)
        rb = F.cd_k_update(b, v0p, 1, 0.1, up)
        assert ra == rb, step
        v0p[:] = (O.bernoulli_f32(10 + step, 0.5, B * V).reshape(B, V))
        v0[:] = v0p
    for x, y in zip(a.get(), b.get()):
        assert np.array_equal(x, y)
    sa, sb = a.last_states(B), b.last_states(B)
    for x, y in zip(sa, sb):
        assert np.array_equal(x, y)


@pytest.mark.parametrize("fused", ["1", "0"])
def test_train_stream_matches_cd_k_calls(gpu, fused, monkeypatch):
    """train_stream (double-buffered host->device staging overlapped with the steps) runs the same
    kernel arithmetic as one cd_k_update call per batch: identical per-step recon and weights"""
    import torch
    from paper_1804_04512_b200 import fastnn as F
    monkeypatch.setenv("B2N_RBM_FUSED", fused)
    S, B, V, H = 5, 100, 784, 500
    v0 = O.bernoulli_f32(3, 0.5, S * B * V).reshape(S * B, V)
    u = O.canonical_f64(5, S * B * H).reshape(S * B, H)
    v0p = torch.empty((S * B, V), dtype=torch.float32, pin_memory=True).numpy()
    up = torch.empty((S * B, H), dtype=torch.float64, pin_memory=True).numpy()
    v0p[:] = v0
    up[:] = u
    a, b = F.Rbm(H, V), F.Rbm(H, V)
    a.init(42)
    b.init(42)
    ra = [F.cd_k_update(a, v0[i * B:(i + 1) * B], 1, 0.1, u[i * B:(i + 1) * B]) for i in range(S)]
    rb = b.train_stream(v0p, up, B, 0.1)
    assert list(rb) == ra
    for x, y in zip(a.get(), b.get()):
        np.testing.assert_array_equal(x, y)
    rc = b.train_stream(v0, u, B, 0.1)  # pageable host buffers: same path, staged copies
    assert np.all(np.isfinite(rc)) and len(rc) == S
