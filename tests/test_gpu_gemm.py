"""tcgen05 GEMM (b2n_gemm) vs the oracle's fastnn gemm (gemm.hpp:225) in all four transpose modes,
including ragged (non-multiple-of-tile) extents and K smaller than one 32-wide K block."""
import numpy as np
import pytest

from conftest import norm_err
from oracle import oracle as O

pytestmark = pytest.mark.gpu

SHAPES = [(100, 500, 784), (37, 53, 29), (128, 128, 32), (100, 10, 250), (10, 251, 100), (500, 785, 100),
          (1, 8, 4), (260, 300, 70)]


@pytest.mark.parametrize("ta", [0, 1])
@pytest.mark.parametrize("tb", [0, 1])
@pytest.mark.parametrize("shape", SHAPES)
def test_gemm_vs_oracle(gpu, ta, tb, shape):
    import torch
    from paper_1804_04512_b200 import fastnn as F
    M, N, K = shape
    rng = np.random.default_rng(M * 7 + N * 3 + K)
    a = rng.standard_normal((K, M) if ta else (M, K)).astype(np.float32)
    b = rng.standard_normal((N, K) if tb else (K, N)).astype(np.float32)
    want = O.gemm(ta, tb, a, b)

    def dev(x):  # fastnn rows are padded to 8 floats (tensor.hpp:142); keep the pad on device
        r, c = x.shape
        cp = (c + 7) // 8 * 8
        t = torch.zeros((r, cp), dtype=torch.float32, device=gpu)
        t[:, :c] = torch.from_numpy(x)
        return t[:, :c]

    got = F.gemm(dev(a), dev(b), bool(ta), bool(tb)).cpu().numpy()
    assert norm_err(got, want) < 1e-5, norm_err(got, want)
    got1 = F.gemm(dev(a), dev(b), bool(ta), bool(tb), precision=F.TF32).cpu().numpy()
    assert norm_err(got1, want) < 5e-3


def test_gemm_hand_product(gpu):
    """test_kernels.cpp:33-41: [[1,2],[3,4]] . [[5,6],[7,8]] = [[19,22],[43,50]]."""
    import torch
    from paper_1804_04512_b200 import fastnn as F
    a = torch.zeros((2, 8), device=gpu)
    b = torch.zeros((2, 8), device=gpu)
    a[:, :2] = torch.tensor([[1.0, 2.0], [3.0, 4.0]])
    b[:, :2] = torch.tensor([[5.0, 6.0], [7.0, 8.0]])
    c = F.gemm(a[:, :2], b[:, :2]).cpu().numpy()
    np.testing.assert_array_equal(c, np.array([[19, 22], [43, 50]], np.float32))
