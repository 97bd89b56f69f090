"""The reference's op-level layer API on the GPU (b2n_op_*, csrc/ops.cu) against the live reference
(oracle/_ref: the unmodified fastnn headers behind ref_shim.cpp) on identical inputs: bit-identical
conv_forward (layers.hpp:132; direct and im2col backends, with and without pad), conv_backward's dx,
gk and gb (layers.hpp:152; gradients accumulate into the incoming tensors), pool_forward /
pool_backward (max with ties, avg), activation_apply / _gradient, softmax and softmax_cross_entropy
(network.hpp:410), plus the reference's error behaviour."""
import ctypes as C

import numpy as np
import pytest

from oracle import oracle as O

pytestmark = pytest.mark.gpu

ref_only = pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built")


def _F():
    from paper_1804_04512_b200 import fastnn as F
    return F


def fp(a):
    return a.ctypes.data_as(C.POINTER(C.c_float))


def rnd(seed, shape, lo=-1.0, hi=1.0):
    return np.random.default_rng(seed).uniform(lo, hi, size=shape).astype(np.float32)


def eq(a, b):
    np.testing.assert_array_equal(np.asarray(a).view(np.uint32) & 0x7FFFFFFF | 0, np.asarray(b).view(np.uint32) & 0x7FFFFFFF | 0)
    np.testing.assert_array_equal(a, b)


CONV_CASES = [  # n, c, h, w, k, kh, kw, pad
    (3, 1, 28, 28, 8, 5, 5, 0),     # MNIST conv0 (im2col backend: h*w >= 784)
    (3, 8, 12, 12, 8, 5, 5, 0),     # MNIST conv1 (direct)
    (2, 3, 32, 32, 12, 5, 5, 0),    # CIFAR conv0
    (2, 12, 14, 14, 12, 5, 5, 0),   # CIFAR conv1
    (2, 16, 16, 16, 16, 3, 3, 1),   # ImageNet-shaped block (padded forward)
    (1, 3, 40, 40, 16, 3, 3, 1),
    (2, 2, 7, 9, 3, 2, 2, 0),       # below 3x3: direct
    (1, 1, 5, 5, 1, 5, 5, 0),
]


@ref_only
@pytest.mark.parametrize("n,c,h,w,k,kh,kw,pad", CONV_CASES)
def test_conv_forward_bit_exact(gpu, n, c, h, w, k, kh, kw, pad):
    F = _F()
    x, ker, b = rnd(1, (n, c, h, w)), rnd(2, (k, c, kh, kw), -0.3, 0.3), rnd(3, (k,))
    y = F.conv_forward(ker, b, x, pad)
    want = np.zeros_like(y)
    O.load("ref").ref_conv_forward(n, c, h, w, k, kh, kw, pad, fp(x), fp(ker), fp(b), fp(want))
    eq(y, want)


@ref_only
@pytest.mark.parametrize("n,c,h,w,k,kh,kw,pad", [cs for cs in CONV_CASES if cs[7] == 0])
def test_conv_backward_bit_exact(gpu, n, c, h, w, k, kh, kw, pad):
    F = _F()
    oh, ow = h - kh + 1, w - kw + 1
    x, ker, dy = rnd(4, (n, c, h, w)), rnd(5, (k, c, kh, kw), -0.3, 0.3), rnd(6, (n, k, oh, ow))
    gk0, gb0 = rnd(7, (k, c, kh, kw), -0.1, 0.1), rnd(8, (k,), -0.1, 0.1)  # accumulate into these
    gk, gb = gk0.copy(), gb0.copy()
    dx = F.conv_backward(ker, x, dy, gk, gb)
    rgk, rgb, rdx = gk0.copy(), gb0.copy(), np.zeros_like(x)
    err = C.create_string_buffer(256)
    assert O.load("ref").ref_conv_backward(n, c, h, w, k, kh, kw, pad, fp(x), fp(ker), fp(dy), fp(rgk), fp(rgb),
                                           fp(rdx), err, 256) == 0, err.value
    eq(dx, rdx)
    eq(gk, rgk)
    eq(gb, rgb)


def test_conv_backward_rejects_padded_forward(gpu):
    F = _F()
    import paper_1804_04512_b200._lib as L
    s = F._ConvShapeC(1, 1, 1, 3, 3, 8, 8, 1)
    z = np.zeros(64, np.float32)
    rc = L.load().b2n_op_conv_backward(0, C.addressof(s), fp(z), fp(z), fp(z), fp(z), fp(z), fp(z))
    assert rc != 0 and b"padded forward has no backward pass" in L.load().b2n_last_error()


@ref_only
@pytest.mark.parametrize("shape", [(2, 3, 8, 6), (5, 4, 4), (2, 2)])
@pytest.mark.parametrize("mode", [0, 1])
def test_pool_bit_exact(gpu, shape, mode):
    F = _F()
    x = np.round(rnd(9, shape) * 4) / 4  # quarter steps: plenty of exact ties inside windows
    y, a = F.pool_forward(mode, x)
    maps = int(np.prod(shape[:-2])) if len(shape) > 2 else 1
    h, w = shape[-2:]
    ry, ra = np.zeros_like(y), np.zeros_like(y)
    O.load("ref").ref_pool_forward(mode, maps, h, w, fp(x), fp(ry), fp(ra))
    eq(y, ry)
    if mode == 0:
        eq(a, ra)
    dy = rnd(10, y.shape)
    dx = F.pool_backward(mode, dy, a)
    rdx = np.zeros_like(dx)
    O.load("ref").ref_pool_backward(mode, maps, h // 2, w // 2, fp(dy), fp(ra if mode == 0 else ry), fp(rdx))
    eq(dx, rdx)


def test_pool_rejects_odd_extents(gpu):
    F = _F()
    with pytest.raises(F.ShapeError, match="spatial extents must be even, got 3x4"):
        F.pool_forward(0, np.zeros((2, 3, 4), np.float32))


@ref_only
@pytest.mark.parametrize("kind", [0, 1])
def test_activation_bit_exact(gpu, kind):
    F = _F()
    x = rnd(11, (4097,), -20.0, 20.0)
    y = F.activation_apply(kind, x)
    ry = np.zeros_like(x)
    O.load("ref").ref_activation_apply(kind, x.size, fp(x), fp(ry))
    eq(y, ry)
    dy = rnd(12, x.shape)
    dx = F.activation_gradient(kind, y, dy)
    rdx = np.zeros_like(x)
    O.load("ref").ref_activation_gradient(kind, x.size, fp(ry), fp(dy), fp(rdx))
    eq(dx, rdx)


@ref_only
@pytest.mark.parametrize("rows,cols", [(100, 10), (16, 1000), (1, 1), (7, 3)])
def test_softmax_and_xent_bit_exact(gpu, rows, cols):
    F = _F()
    x = rnd(13, (rows, cols), -8.0, 8.0)
    p = F.softmax(x)
    rp = np.zeros_like(x)
    O.load("ref").ref_softmax(rows, cols, fp(x), fp(rp))
    eq(p, rp)
    lab = np.random.default_rng(14).integers(0, cols, rows)
    y = np.eye(cols, dtype=np.float32)[lab]
    loss, g = F.softmax_cross_entropy(p, y)
    rg, rl = np.zeros_like(p), C.c_double()
    err = C.create_string_buffer(256)
    assert O.load("ref").ref_softmax_cross_entropy(rows, cols, fp(rp), fp(y), fp(rg), C.byref(rl), err, 256) == 0
    eq(g, rg)
    assert abs(loss - rl.value) <= 1e-13 * max(1.0, abs(rl.value))


def test_xent_rejects_non_one_hot(gpu):
    F = _F()
    p = np.full((2, 3), 1 / 3, np.float32)
    y = np.array([[1, 0, 0], [0, 0.5, 0]], np.float32)
    with pytest.raises(F.LabelError, match="labels must be one-hot; row 1"):
        F.softmax_cross_entropy(p, y)
