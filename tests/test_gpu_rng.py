"""The reference's Bernoulli stream generated on the device (csrc/mt19937.cuh): std::mt19937 +
generate_canonical<double,53> (energy.hpp:53-71 via std::bernoulli_distribution) bit for bit, the
generator state advanced exactly as libstdc++ leaves it, and every sampling step (CD-1, CD-k, the
streamed loop, the CRBM, the DBN) identical whether the draws come from the device generator or
are drawn on the host and supplied."""
import numpy as np
import pytest

from oracle import oracle as O

pytestmark = pytest.mark.gpu


def _F():
    from paper_1804_04512_b200 import fastnn as F
    return F


@pytest.mark.parametrize("skip,n", [(0, 1_000_000), (77, 312), (0, 0), (1, 311), (623, 1), (5, 2_000_001),
                                    (0, 312), (100, 262)])
def test_draws_bit_exact(gpu, skip, n):
    F = _F()
    host, dev = F.Mt19937(1234), F.Mt19937(1234)
    if skip:  # leave the generator mid-block (odd positions included)
        host._rs.randint(0, 2 ** 32, size=skip, dtype=np.uint64)
        dev._rs.randint(0, 2 ** 32, size=skip, dtype=np.uint64)
    got = F.mt19937_draw(dev, n)
    want = host.canonical(n)
    np.testing.assert_array_equal(got.view(np.uint64), want.view(np.uint64))
    np.testing.assert_array_equal(dev.state(), host.state())
    if n:
        assert got.min() >= 0.0 and got.max() < 1.0


def test_draws_match_std_mt19937(gpu):
    """against the C++ standard library itself (the oracle's std::mt19937 + generate_canonical)"""
    F = _F()
    got = F.mt19937_draw(F.Mt19937(5), 50_000)
    np.testing.assert_array_equal(got, O.canonical_f64(5, 50_000))


def test_consecutive_draws_continue_the_stream(gpu):
    F = _F()
    host, dev = F.Mt19937(9), F.Mt19937(9)
    parts = [F.mt19937_draw(dev, m) for m in (1, 623, 624, 5000, 3)]
    np.testing.assert_array_equal(np.concatenate(parts), host.canonical(sum(p.size for p in parts)))


def _same_params(a, b):
    for x, y in zip(a.get(), b.get()):
        np.testing.assert_array_equal(x, y)


@pytest.mark.parametrize("B,H,V,k", [(100, 500, 784, 1), (37, 64, 100, 1), (20, 48, 96, 2), (130, 64, 100, 1)])
def test_cd_k_device_draws_equal_supplied(gpu, B, H, V, k):
    F = _F()
    r1, r2 = F.Rbm(H, V), F.Rbm(H, V)
    r1.init(42)
    r2.init(42)
    ga, gb = F.Mt19937(5), F.Mt19937(5)
    for step in range(3):
        v0 = O.bernoulli_f32(3 + step, 0.5, B * V).reshape(B, V)
        ra = F.cd_k_update(r1, v0, k, 0.1, ga)              # device generator
        rb = F.cd_k_update(r2, v0, k, 0.1, gb.canonical(k * B * H))  # host draws, supplied
        assert ra == rb
        np.testing.assert_array_equal(r1.last_states(B)[1], r2.last_states(B)[1])
    _same_params(r1, r2)
    np.testing.assert_array_equal(ga.state(), gb.state())


def test_cd1_pinned_direct_path_device_draws(gpu):
    """the fused step's zero-copy launch (pinned v0) with the draws from the device generator"""
    import torch
    F = _F()
    B, H, V = 100, 500, 784
    r1, r2 = F.Rbm(H, V), F.Rbm(H, V)
    r1.init(1)
    r2.init(1)
    ga, gb = F.Mt19937(77), F.Mt19937(77)
    v0 = torch.from_numpy(O.bernoulli_f32(4, 0.5, B * V).reshape(B, V)).pin_memory()
    for _ in range(2):
        ra = F.cd_k_update(r1, v0.numpy(), 1, 0.05, ga)
        rb = F.cd_k_update(r2, v0.numpy(), 1, 0.05, gb.canonical(B * H))
        assert ra == rb
    _same_params(r1, r2)
    np.testing.assert_array_equal(ga.state(), gb.state())


@pytest.mark.parametrize("steps,B,H,V", [(7, 100, 500, 784), (1, 100, 500, 784), (4, 13, 500, 784),
                                         (37, 100, 500, 784), (25, 4, 8, 16), (12, 7, 40, 24)])
def test_train_stream_device_draws(gpu, steps, B, H, V):
    """train_stream generates each step's draws with its start state found by jump-ahead (several steps
    in flight): every recon, the parameters and the final generator state equal host draws supplied in
    order -- including long streams and steps whose draws stay inside one 624-word block"""
    F = _F()
    r1, r2 = F.Rbm(H, V), F.Rbm(H, V)
    r1.init(3)
    r2.init(3)
    v = O.bernoulli_f32(8, 0.4, steps * B * V).reshape(steps * B, V)
    ga, gb = F.Mt19937(21), F.Mt19937(21)
    rec_a = r1.train_stream(v, ga, B, 0.1)
    rec_b = r2.train_stream(v, gb.canonical(steps * B * H), B, 0.1)
    np.testing.assert_array_equal(rec_a, rec_b)
    _same_params(r1, r2)
    np.testing.assert_array_equal(ga.state(), gb.state())
    # and the generator continues correctly into a per-call step
    v1 = O.bernoulli_f32(9, 0.4, B * V).reshape(B, V)
    assert F.cd_k_update(r1, v1, 1, 0.1, ga) == F.cd_k_update(r2, v1, 1, 0.1, gb.canonical(B * H))
    np.testing.assert_array_equal(ga.state(), gb.state())


def test_crbm_device_draws_equal_supplied(gpu):
    F = _F()
    B = 100
    m1, m2 = F.Crbm(1, 28, 28, 12, 5, 5), F.Crbm(1, 28, 28, 12, 5, 5)
    m1.init(42)
    m2.init(42)
    ga, gb = F.Mt19937(5), F.Mt19937(5)
    for step in range(2):
        v0 = O.bernoulli_f32(3 + step, 0.5, B * 784).reshape(B, 1, 28, 28)
        ra = F.crbm_cd_update(m1, v0, 0.1, ga)
        rb = F.crbm_cd_update(m2, v0, 0.1, gb.canonical(B * 12 * 24 * 24))
        assert ra == rb
    _same_params(m1, m2)
    np.testing.assert_array_equal(ga.state(), gb.state())


@pytest.mark.parametrize("steps,B", [(6, 100), (1, 100), (5, 17)])
def test_crbm_train_stream_device_draws(gpu, steps, B):
    """the CRBM's streamed loop with 16 generators in flight (jump-ahead start states) equals the
    per-call loop with the host's draws: every recon, the parameters, the generator state"""
    F = _F()
    m1, m2 = F.Crbm(1, 28, 28, 12, 5, 5), F.Crbm(1, 28, 28, 12, 5, 5)
    m1.init(4)
    m2.init(4)
    v = O.bernoulli_f32(12, 0.5, steps * B * 784).reshape(steps * B, 1, 28, 28)
    ga, gb = F.Mt19937(31), F.Mt19937(31)
    rec = m1.train_stream(v, ga, B, 0.1)
    want = [F.crbm_cd_update(m2, v[i * B:(i + 1) * B], 0.1, gb.canonical(B * 12 * 24 * 24)) for i in range(steps)]
    np.testing.assert_array_equal(rec, np.array(want))
    _same_params(m1, m2)
    np.testing.assert_array_equal(ga.state(), gb.state())


def test_dbn_device_draws_equal_host(gpu):
    F = _F()
    data = O.bernoulli_f32(2, 0.5, 250 * 64).reshape(250, 64)

    def stack():
        s = [F.Rbm(48, 64), F.Rbm(32, 48)]
        s[0].init(1)
        s[1].init(2)
        return s

    s1, s2 = stack(), stack()
    ga, gb = F.Mt19937(6), F.Mt19937(6)
    rep_a = F.dbn_pretrain(s1, data, 2, 0.1, 40, ga)
    rep_b = F.dbn_pretrain(s2, data, 2, 0.1, 40, gb, host_draws=True)
    assert rep_a.recon == rep_b.recon
    for a, b in zip(s1, s2):
        _same_params(a, b)
    np.testing.assert_array_equal(ga.state(), gb.state())


@pytest.mark.parametrize("skip", [77, 623, 1])
def test_crbm_train_stream_mid_block(gpu, skip):
    """the CRBM's streamed loop (691,200 draws per step, 24 generators from jumps) started mid-block --
    odd and last-word positions -- equals the host's draws in order"""
    F = _F()
    B, steps = 100, 3
    m1, m2 = F.Crbm(1, 28, 28, 12, 5, 5), F.Crbm(1, 28, 28, 12, 5, 5)
    m1.init(8)
    m2.init(8)
    v = O.bernoulli_f32(14, 0.5, steps * B * 784).reshape(steps * B, 1, 28, 28)
    ga, gb = F.Mt19937(41), F.Mt19937(41)
    ga._rs.randint(0, 2 ** 32, size=skip, dtype=np.uint64)
    gb._rs.randint(0, 2 ** 32, size=skip, dtype=np.uint64)
    rec = m1.train_stream(v, ga, B, 0.1)
    want = [F.crbm_cd_update(m2, v[i * B:(i + 1) * B], 0.1, gb.canonical(B * 12 * 24 * 24)) for i in range(steps)]
    np.testing.assert_array_equal(rec, np.array(want))
    _same_params(m1, m2)
    np.testing.assert_array_equal(ga.state(), gb.state())
