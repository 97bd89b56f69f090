"""ctypes access to the parity checker (TEST INFRASTRUCTURE ONLY).

Only tests/, __graft_entry__.smoke() and bench.py (cpu_baseline leg and --impl reference) import
this module. It loads
  * oracle/_build/liboracle.so  -- the C++ restatement (oracle/fastnn_oracle.cpp), built on demand
                                   with `make -C oracle` (g++ is on every box), and
  * oracle/_ref/libfastnn_ref.so -- the reference headers compiled behind oracle/ref_shim.cpp
                                   (only buildable where /root/reference exists; optional).
Both expose the same network / RBM / op entry points so a test can run either side.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
ORACLE_SO = HERE / "_build" / "liboracle.so"
REF_SO = HERE / "_ref" / "libfastnn_ref.so"

# LayerDesc kinds, same numbering as fastnn::LayerDesc::Kind (network.hpp:195) and include/b200nn.h
DENSE, CONV, MAXPOOL, SIGMOID, RELU, SOFTMAX, DROPOUT, BATCHNORM, FLATTEN = range(9)


class LayerDescC(C.Structure):
    _fields_ = [("kind", C.c_int), ("in_", C.c_longlong), ("out", C.c_longlong), ("k", C.c_longlong),
                ("kh", C.c_longlong), ("kw", C.c_longlong), ("pad", C.c_longlong), ("p", C.c_float)]


def build() -> None:
    subprocess.run(["make", "-s", "-C", str(HERE)], check=True)


_lib_cache: dict[str, C.CDLL] = {}

_F = C.POINTER(C.c_float)
_D = C.POINTER(C.c_double)
_I = C.POINTER(C.c_int)
_LL = C.POINTER(C.c_longlong)


def _declare(lib: C.CDLL, prefix: str) -> None:
    p = prefix
    f = getattr(lib, f"{p}_net_create")
    if p == "orc":
        f.argtypes = [C.c_int, _LL, C.POINTER(LayerDescC), C.c_int, C.c_float, C.c_float, C.c_float, C.c_uint,
                      C.c_char_p, C.c_int]
    else:
        f.argtypes = [C.c_int, _LL, C.POINTER(LayerDescC), C.c_int, C.c_float, C.c_float, C.c_float, C.c_uint,
                      C.c_longlong, C.c_char_p, C.c_int]
    f.restype = C.c_void_p
    getattr(lib, f"{p}_net_destroy").argtypes = [C.c_void_p]
    getattr(lib, f"{p}_net_num_params").argtypes = [C.c_void_p]
    getattr(lib, f"{p}_net_param_size").argtypes = [C.c_void_p, C.c_int]
    getattr(lib, f"{p}_net_param_size").restype = C.c_longlong
    getattr(lib, f"{p}_net_get").argtypes = [C.c_void_p, C.c_int, C.c_int, _F]
    getattr(lib, f"{p}_net_set").argtypes = [C.c_void_p, C.c_int, C.c_int, _F]
    getattr(lib, f"{p}_net_apply").argtypes = [C.c_void_p]
    getattr(lib, f"{p}_net_train_minibatch").argtypes = [C.c_void_p, _F, _I, C.c_longlong]
    getattr(lib, f"{p}_net_train_minibatch").restype = C.c_double
    getattr(lib, f"{p}_net_forward").argtypes = [C.c_void_p, _F, C.c_longlong, _F, _I]
    fb = getattr(lib, f"{p}_net_forward_backward")
    if p == "orc":
        fb.argtypes = [C.c_void_p, _F, _I, C.c_longlong, C.c_longlong, _F]
    else:
        fb.argtypes = [C.c_void_p, _F, _I, C.c_longlong, _F]
    fb.restype = C.c_double
    g = getattr(lib, f"{p}_gemm")
    g.argtypes = [C.c_int, C.c_int, _F, _F, _F, C.c_longlong, C.c_longlong, C.c_longlong]
    getattr(lib, f"{p}_sgd_momentum_step").argtypes = [_F, _F, _F, C.c_longlong, C.c_float, C.c_float, C.c_float]
    getattr(lib, f"{p}_net_set_optimizer").argtypes = [C.c_void_p, C.c_int]
    getattr(lib, f"{p}_batch_order").argtypes = [C.c_longlong, C.c_uint, C.c_int, _LL]
    getattr(lib, f"{p}_net_fit").argtypes = [C.c_void_p, _F, _I, C.c_longlong, C.c_longlong, C.c_uint, C.c_int,
                                             _D, _D]
    getattr(lib, f"{p}_net_evaluate").argtypes = [C.c_void_p, _F, _I, C.c_longlong, C.c_longlong]
    getattr(lib, f"{p}_net_evaluate").restype = C.c_double
    getattr(lib, f"{p}_rbm_init").argtypes = [C.c_longlong, C.c_longlong, C.c_uint, _F]
    if p == "orc":
        lib.orc_net_set_hparams.argtypes = [C.c_void_p, C.c_float, C.c_float, C.c_float]
        lib.orc_rbm_cd1.argtypes = [C.c_longlong, C.c_longlong, _F, _F, _F, _F, C.c_longlong, C.c_longlong,
                                    C.c_float, _D, _F, _F, _F, _F, _F, _F, _F]
        lib.orc_rbm_cd1.restype = C.c_double
        lib.orc_rbm_cdk.argtypes = [C.c_longlong, C.c_longlong, _F, _F, _F, _F, C.c_longlong, C.c_longlong,
                                    C.c_int, C.c_float, _D, _F, _F, _F, _F, _F, _F, _F, _F]
        lib.orc_rbm_cdk.restype = C.c_double
        lib.orc_conv_forward.argtypes = [_F, C.c_longlong, C.c_longlong, C.c_longlong, C.c_longlong, _F, _F,
                                         C.c_longlong, C.c_longlong, C.c_longlong, C.c_longlong, _F]
        lib.orc_conv_backward.argtypes = [_F, C.c_longlong, C.c_longlong, C.c_longlong, C.c_longlong, _F,
                                          C.c_longlong, C.c_longlong, C.c_longlong, C.c_longlong, _F, _F, _F, _F]
        lib.orc_uniform_f32.argtypes = [C.c_uint, C.c_float, C.c_float, C.c_longlong, _F]
        lib.orc_rbm_transform_up.argtypes = [C.c_longlong, C.c_longlong, _F, _F, _F, C.c_longlong, _F]
        lib.orc_canonical_f64.argtypes = [C.c_uint, C.c_longlong, _D]
        lib.orc_bernoulli_f32.argtypes = [C.c_uint, C.c_double, C.c_longlong, _F]
        lib.orc_uniform_int.argtypes = [C.c_uint, C.c_int, C.c_int, C.c_longlong, _I]
        lib.orc_crbm_cd1.argtypes = [C.c_longlong] * 6 + [_F, _F, _F, _F, C.c_longlong, C.c_longlong, C.c_float,
                                                          _D, _F, _F, _F, _F, _F, _F, _F]
        lib.orc_crbm_cd1.restype = C.c_double
        lib.orc_crbm_init.argtypes = [C.c_longlong] * 4 + [C.c_uint, _F]
        lib.orc_set_exact_sums.argtypes = [C.c_int]
    else:
        lib.ref_cd_k.argtypes = [C.c_longlong, C.c_longlong, _F, _F, _F, _F, C.c_longlong, C.c_int, C.c_float,
                                 C.c_uint]
        lib.ref_cd_k.restype = C.c_double
        lib.ref_make_batch.argtypes = [C.c_void_p, _F, _I, C.c_longlong]
        lib.ref_make_batch.restype = C.c_void_p
        lib.ref_free_batch.argtypes = [C.c_void_p]
        lib.ref_net_train_prepared.argtypes = [C.c_void_p, C.c_void_p]
        lib.ref_net_train_prepared.restype = C.c_double
        lib.ref_rbm_create.argtypes = [C.c_longlong, C.c_longlong, C.c_uint, _F, C.c_longlong, C.c_uint]
        lib.ref_rbm_create.restype = C.c_void_p
        lib.ref_rbm_step.argtypes = [C.c_void_p, C.c_float]
        lib.ref_rbm_step.restype = C.c_double
        lib.ref_rbm_destroy.argtypes = [C.c_void_p]
        lib.ref_save_network.argtypes = [C.c_void_p, C.c_char_p, C.c_char_p, C.c_int]
        lib.ref_load_network.argtypes = [C.c_void_p, C.c_char_p, C.c_char_p, C.c_int]
        lib.ref_dbn_pretrain.argtypes = [C.c_int, _LL, _LL, _F, _F, _F, _F, C.c_longlong, C.c_int, C.c_float,
                                         C.c_longlong, C.c_uint, _D, C.c_char_p, C.c_int]
        lib.ref_set_threads.argtypes = [C.c_int]
        lib.ref_crbm_cd.argtypes = [C.c_longlong] * 6 + [_F, _F, _F, _F, C.c_longlong, C.c_float, C.c_uint]
        lib.ref_crbm_cd.restype = C.c_double
        lib.ref_crbm_init.argtypes = [C.c_longlong] * 6 + [C.c_uint, _F]
        lib.ref_crbm_create.argtypes = [C.c_longlong] * 6 + [C.c_uint, _F, C.c_longlong, C.c_uint]
        lib.ref_crbm_create.restype = C.c_void_p
        lib.ref_crbm_step.argtypes = [C.c_void_p, C.c_float]
        lib.ref_crbm_step.restype = C.c_double
        lib.ref_crbm_destroy.argtypes = [C.c_void_p]
        lib.ref_thread_count.restype = C.c_int
        # the reference's op-level layer API (b2n_op_* parity)
        LL = C.c_longlong
        lib.ref_conv_forward.argtypes = [LL] * 8 + [_F, _F, _F, _F]
        lib.ref_conv_backward.argtypes = [LL] * 8 + [_F, _F, _F, _F, _F, _F, C.c_char_p, C.c_int]
        lib.ref_conv_backward.restype = C.c_int
        lib.ref_pool_forward.argtypes = [C.c_int, LL, LL, LL, _F, _F, _F]
        lib.ref_pool_backward.argtypes = [C.c_int, LL, LL, LL, _F, _F, _F]
        lib.ref_softmax.argtypes = [LL, LL, _F, _F]
        lib.ref_softmax_cross_entropy.argtypes = [LL, LL, _F, _F, _F, _D, C.c_char_p, C.c_int]
        lib.ref_softmax_cross_entropy.restype = C.c_int
        lib.ref_activation_apply.argtypes = [C.c_int, LL, _F, _F]
        lib.ref_activation_gradient.argtypes = [C.c_int, LL, _F, _F, _F]


def load(which: str = "oracle") -> C.CDLL:
    """which = 'oracle' (restatement, always available) or 'ref' (compiled reference, optional)."""
    if which in _lib_cache:
        return _lib_cache[which]
    path = ORACLE_SO if which == "oracle" else REF_SO
    if not path.exists() and which == "oracle":
        build()
    if not path.exists():
        raise FileNotFoundError(f"{path} not built (needs /root/reference at build time)")
    lib = C.CDLL(str(path))
    _declare(lib, "orc" if which == "oracle" else "ref")
    _lib_cache[which] = lib
    return lib


def set_exact_sums(on: bool) -> None:
    """Restatement only: conv kernel / bias gradient sums in double (the float64 truth of the
    reference's own summands), see g_exact_sums in fastnn_oracle.cpp."""
    load("oracle").orc_set_exact_sums(1 if on else 0)


def ref_available() -> bool:
    try:
        load("ref")
        return True
    except (FileNotFoundError, OSError):
        return False


def fptr(a: np.ndarray):
    assert a.dtype == np.float32 and a.flags.c_contiguous
    return a.ctypes.data_as(_F)


def dptr(a: np.ndarray):
    assert a.dtype == np.float64 and a.flags.c_contiguous
    return a.ctypes.data_as(_D)


def iptr(a: np.ndarray):
    assert a.dtype == np.int32 and a.flags.c_contiguous
    return a.ctypes.data_as(_I)


def layers_c(layers: list[dict]):
    arr = (LayerDescC * len(layers))()
    for i, d in enumerate(layers):
        arr[i].kind = d["kind"]
        arr[i].in_ = d.get("in", 0)
        arr[i].out = d.get("out", 0)
        arr[i].k = d.get("k", 0)
        arr[i].kh = d.get("kh", 0)
        arr[i].kw = d.get("kw", 0)
        arr[i].pad = d.get("pad", 0)
        arr[i].p = d.get("p", 0.0)
    return arr


class Net:
    """A network on one side ('oracle' or 'ref'); mirrors fastnn::Network's step surface."""

    def __init__(self, spec: dict, which: str = "oracle"):
        self.which = which
        self.lib = load(which)
        self.p = "orc" if which == "oracle" else "ref"
        inp = (C.c_longlong * len(spec["input"]))(*spec["input"])
        arr = layers_c(spec["layers"])
        err = C.create_string_buffer(512)
        args = [len(spec["input"]), inp, arr, len(spec["layers"]), spec.get("lr", 0.1), spec.get("momentum", 0.9),
                spec.get("weight_decay", 0.0), spec.get("seed", 42)]
        if which == "ref":
            args.append(spec.get("batch_size", 100))
        h = getattr(self.lib, f"{self.p}_net_create")(*args, err, 512)
        if not h:
            raise ValueError(err.value.decode())
        self.h = h
        self.classes = [d for d in spec["layers"] if d["kind"] == DENSE][-1]["out"]
        self.input = list(spec["input"])
        if spec.get("optimizer", 0):
            getattr(self.lib, f"{self.p}_net_set_optimizer")(self.h, spec["optimizer"])

    def __del__(self):
        if getattr(self, "h", None):
            getattr(self.lib, f"{self.p}_net_destroy")(self.h)
            self.h = None

    def num_params(self) -> int:
        return getattr(self.lib, f"{self.p}_net_num_params")(self.h)

    def get(self, idx: int, which: int = 0) -> np.ndarray:
        n = getattr(self.lib, f"{self.p}_net_param_size")(self.h, idx)
        out = np.zeros(n, np.float32)
        getattr(self.lib, f"{self.p}_net_get")(self.h, idx, which, fptr(out))
        return out

    def set(self, idx: int, values: np.ndarray, which: int = 0) -> None:
        v = np.ascontiguousarray(values, np.float32).ravel()
        getattr(self.lib, f"{self.p}_net_set")(self.h, idx, which, fptr(v))

    def params(self, which: int = 0) -> list[np.ndarray]:
        return [self.get(i, which) for i in range(self.num_params())]

    def train_minibatch(self, x: np.ndarray, labels: np.ndarray) -> float:
        x = np.ascontiguousarray(x, np.float32)
        labels = np.ascontiguousarray(labels, np.int32)
        return getattr(self.lib, f"{self.p}_net_train_minibatch")(self.h, fptr(x), iptr(labels), labels.shape[0])

    def forward_backward(self, x, labels, b_global=None, probs=None):
        x = np.ascontiguousarray(x, np.float32)
        labels = np.ascontiguousarray(labels, np.int32)
        B = labels.shape[0]
        pp = fptr(probs) if probs is not None else None
        if self.p == "orc":
            return self.lib.orc_net_forward_backward(self.h, fptr(x), iptr(labels), B, b_global or B, pp)
        assert b_global in (None, B)
        return self.lib.ref_net_forward_backward(self.h, fptr(x), iptr(labels), B, pp)

    def apply(self) -> None:
        getattr(self.lib, f"{self.p}_net_apply")(self.h)

    def forward(self, x: np.ndarray):
        x = np.ascontiguousarray(x, np.float32)
        B = x.shape[0]
        probs = np.zeros((B, self.classes), np.float32)
        am = np.zeros(B, np.int32)
        getattr(self.lib, f"{self.p}_net_forward")(self.h, fptr(x), B, fptr(probs), iptr(am))
        return probs, am


    def fit(self, x: np.ndarray, labels: np.ndarray, batch: int, seed: int, epochs: int):
        """fit (network.hpp:488-511): per-epoch (loss, train accuracy)"""
        x = np.ascontiguousarray(x, np.float32)
        labels = np.ascontiguousarray(labels, np.int32)
        loss = np.zeros(epochs, np.float64)
        acc = np.zeros(epochs, np.float64)
        getattr(self.lib, f"{self.p}_net_fit")(self.h, fptr(x), iptr(labels), labels.shape[0], batch, seed, epochs,
                                               dptr(loss), dptr(acc))
        return loss, acc

    def evaluate(self, x: np.ndarray, labels: np.ndarray, batch: int) -> float:
        x = np.ascontiguousarray(x, np.float32)
        labels = np.ascontiguousarray(labels, np.int32)
        return getattr(self.lib, f"{self.p}_net_evaluate")(self.h, fptr(x), iptr(labels), labels.shape[0], batch)


def rbm_transform_up(W, bh, data):
    """rbm_transform_up (energy.hpp:122-126): sigmoid(data . W^T + bh)"""
    W = np.ascontiguousarray(W, np.float32)
    bh = np.ascontiguousarray(bh, np.float32)
    data = np.ascontiguousarray(data, np.float32)
    H, V = W.shape
    out = np.zeros((data.shape[0], H), np.float32)
    load().orc_rbm_transform_up(H, V, fptr(W), fptr(bh), fptr(data), data.shape[0], fptr(out))
    return out


def dbn_pretrain(stack, data, epochs, lr, batch, seed):
    """dbn_pretrain (energy.hpp:208-240) restated over the oracle's CD-1: each layer trains with CD-1
    on the previous layer's hidden means, batches in file order, ONE std::mt19937(seed) stream of
    generate_canonical<double,53> draws across layers, epochs and batches (B x H per step).
    stack = [(W, bv, bh)] (copied); returns (trained stack, recon[layer][epoch])."""
    stack = [(np.array(W, np.float32), np.array(bv, np.float32), np.array(bh, np.float32)) for W, bv, bh in stack]
    n = data.shape[0]
    draws = sum(epochs * n * W.shape[0] for W, _, _ in stack)
    u = canonical_f64(seed, draws)
    pos = 0
    cur = np.ascontiguousarray(data, np.float32)
    recon = []
    for li, (W, bv, bh) in enumerate(stack):
        H = W.shape[0]
        rl = []
        for _ in range(epochs):
            total, nb = 0.0, 0
            for lo in range(0, n, batch):
                hi = min(lo + batch, n)
                r, W, bv, bh, _ = rbm_cd1(W, bv, bh, cur[lo:hi], lr, u[pos:pos + (hi - lo) * H].reshape(hi - lo, H))
                pos += (hi - lo) * H
                total += r
                nb += 1
            rl.append(total / nb)
        stack[li] = (W, bv, bh)
        recon.append(rl)
        if li + 1 < len(stack):
            cur = rbm_transform_up(W, bh, cur)
    return stack, recon


def ref_dbn_pretrain(stack, data, epochs, lr, batch, seed):
    """the reference's own dbn_pretrain (needs oracle/_ref); same contract as dbn_pretrain()"""
    lib = load("ref")
    vis = np.array([w.shape[1] for w, _, _ in stack], np.int64)
    hid = np.array([w.shape[0] for w, _, _ in stack], np.int64)
    W = np.concatenate([np.ravel(w) for w, _, _ in stack]).astype(np.float32)
    bv = np.concatenate([np.ravel(b) for _, b, _ in stack]).astype(np.float32)
    bh = np.concatenate([np.ravel(b) for _, _, b in stack]).astype(np.float32)
    data = np.ascontiguousarray(data, np.float32)
    rec = np.zeros(len(stack) * epochs, np.float64)
    err = C.create_string_buffer(512)
    if lib.ref_dbn_pretrain(len(stack), vis.ctypes.data_as(_LL), hid.ctypes.data_as(_LL), fptr(W), fptr(bv), fptr(bh), fptr(data), data.shape[0],
                            epochs, lr, batch, seed, dptr(rec), err, 512):
        raise RuntimeError(err.value.decode())
    out, ow, ov, oh = [], 0, 0, 0
    for l in range(len(stack)):
        V, H = int(vis[l]), int(hid[l])
        out.append((W[ow:ow + H * V].reshape(H, V), bv[ov:ov + V], bh[oh:oh + H]))
        ow, ov, oh = ow + H * V, ov + V, oh + H
    return out, rec.reshape(len(stack), epochs).tolist()


def ref_checkpoint(net: "Net", path: str, load: bool = False) -> str:
    """the reference's save_network / load_network on a 'ref' net; returns '' or the error text"""
    assert net.which == "ref"
    err = C.create_string_buffer(512)
    fn = net.lib.ref_load_network if load else net.lib.ref_save_network
    return "" if fn(net.h, str(path).encode(), err, 512) == 0 else err.value.decode()


def batch_order(n: int, seed: int, epoch: int, which: str = "oracle") -> np.ndarray:
    """BatchIterator's sample order (data.hpp:224-238) for epoch `epoch`"""
    lib = load(which)
    out = np.zeros(n, np.int64)
    getattr(lib, f"{'orc' if which == 'oracle' else 'ref'}_batch_order")(n, seed, epoch, out.ctypes.data_as(_LL))
    return out


def gemm(ta: bool, tb: bool, a: np.ndarray, b: np.ndarray, which: str = "oracle") -> np.ndarray:
    lib = load(which)
    a = np.ascontiguousarray(a, np.float32)
    b = np.ascontiguousarray(b, np.float32)
    M = a.shape[1] if ta else a.shape[0]
    K = a.shape[0] if ta else a.shape[1]
    N = b.shape[0] if tb else b.shape[1]
    c = np.zeros((M, N), np.float32)
    getattr(lib, "orc_gemm" if which == "oracle" else "ref_gemm")(int(ta), int(tb), fptr(a), fptr(b), fptr(c), M, N, K)
    return c


def rbm_cd1(W, bv, bh, v0, lr, u, b_global=None, deltas=False):
    """Oracle CD-1 with supplied uniforms u[B][H]. Returns (recon, W, bv, bh, extras)."""
    lib = load("oracle")
    W = np.array(W, np.float32, copy=True, order="C")
    bv = np.array(bv, np.float32, copy=True)
    bh = np.array(bh, np.float32, copy=True)
    v0 = np.ascontiguousarray(v0, np.float32)
    u = np.ascontiguousarray(u, np.float64)
    H, V = W.shape
    B = v0.shape[0]
    h0 = np.zeros((B, H), np.float32)
    hs = np.zeros((B, H), np.float32)
    v1 = np.zeros((B, V), np.float32)
    h1 = np.zeros((B, H), np.float32)
    dW = np.zeros((H, V), np.float32) if deltas else None
    dbh = np.zeros(H, np.float32) if deltas else None
    dbv = np.zeros(V, np.float32) if deltas else None
    recon = lib.orc_rbm_cd1(H, V, fptr(W), fptr(bv), fptr(bh), fptr(v0), B, b_global or B, lr, dptr(u), fptr(h0),
                            fptr(hs), fptr(v1), fptr(h1), fptr(dW) if deltas else None,
                            fptr(dbh) if deltas else None, fptr(dbv) if deltas else None)
    extra = dict(h0=h0, hs=hs, v1=v1, h1=h1, dW=dW, dbh=dbh, dbv=dbv)
    return recon, W, bv, bh, extra


def rbm_cdk(W, bv, bh, v0, k, lr, u, b_global=None):
    """Oracle CD-k (energy.hpp:131-171) with supplied uniforms u[k][B][H] (the draw order of the
    reference's std::mt19937 stream). Returns (recon, W, bv, bh, extras); extras["hs"] is the LAST
    sampled hidden state, "v1" the step-1 visible means, "vk" the final ones, "h1" = hk."""
    lib = load("oracle")
    W = np.array(W, np.float32, copy=True, order="C")
    bv = np.array(bv, np.float32, copy=True)
    bh = np.array(bh, np.float32, copy=True)
    v0 = np.ascontiguousarray(v0, np.float32)
    u = np.ascontiguousarray(u, np.float64).ravel()
    H, V = W.shape
    B = v0.shape[0]
    assert u.size >= k * B * H
    h0, hs, h1 = (np.zeros((B, H), np.float32) for _ in range(3))
    v1, vk = np.zeros((B, V), np.float32), np.zeros((B, V), np.float32)
    recon = lib.orc_rbm_cdk(H, V, fptr(W), fptr(bv), fptr(bh), fptr(v0), B, b_global or B, k, lr, dptr(u), fptr(h0),
                            fptr(hs), fptr(v1), fptr(h1), fptr(vk), None, None, None)
    return recon, W, bv, bh, dict(h0=h0, hs=hs, v1=v1, h1=h1, vk=vk)


def force_samples(u, hs):
    """uniforms that make `u < p` reproduce the given binary samples for any p in (0, 1]: 0 where
    hs = 1, 2 where hs = 0 (re-running the oracle on a kernel's own samples)."""
    return np.where(np.asarray(hs).reshape(np.shape(u)) > 0.5, 0.0, 2.0)


def ref_cd_k(W, bv, bh, v0, k, lr, seed):
    lib = load("ref")
    W = np.array(W, np.float32, copy=True, order="C")
    bv = np.array(bv, np.float32, copy=True)
    bh = np.array(bh, np.float32, copy=True)
    v0 = np.ascontiguousarray(v0, np.float32)
    H, V = W.shape
    recon = lib.ref_cd_k(H, V, fptr(W), fptr(bv), fptr(bh), fptr(v0), v0.shape[0], k, lr, seed)
    return recon, W, bv, bh


def rbm_init(H: int, V: int, seed: int, which: str = "oracle") -> np.ndarray:
    lib = load(which)
    W = np.zeros((H, V), np.float32)
    getattr(lib, "orc_rbm_init" if which == "oracle" else "ref_rbm_init")(H, V, seed, fptr(W))
    return W


def crbm_cd1(ker, bv, bh, v0, lr, u, b_global=None, deltas=False):
    """Oracle CRBM CD-1 (crbm_cd_update, energy.hpp:333-376) with supplied uniforms u[B][k][oh][ow].
    ker (k,c,kh,kw), v0 (B,c,h,w). Returns (recon, ker, bv, bh, extras)."""
    lib = load("oracle")
    ker = np.array(ker, np.float32, copy=True, order="C")
    bv = np.array(bv, np.float32, copy=True)
    bh = np.array(bh, np.float32, copy=True)
    v0 = np.ascontiguousarray(v0, np.float32)
    u = np.ascontiguousarray(u, np.float64)
    k, c, kh, kw = ker.shape
    B, _, h, w = v0.shape
    oh, ow = h - kh + 1, w - kw + 1
    h0 = np.zeros((B, k, oh, ow), np.float32)
    hs, h1 = np.zeros_like(h0), np.zeros_like(h0)
    v1 = np.zeros_like(v0)
    dk = np.zeros_like(ker) if deltas else None
    dbh = np.zeros(k, np.float32) if deltas else None
    dbv = np.zeros(c, np.float32) if deltas else None
    recon = lib.orc_crbm_cd1(c, h, w, k, kh, kw, fptr(ker), fptr(bv), fptr(bh), fptr(v0), B, b_global or B, lr,
                             dptr(u), fptr(h0), fptr(hs), fptr(v1), fptr(h1), fptr(dk) if deltas else None,
                             fptr(dbh) if deltas else None, fptr(dbv) if deltas else None)
    return recon, ker, bv, bh, dict(h0=h0, hs=hs, v1=v1, h1=h1, dker=dk, dbh=dbh, dbv=dbv)


def ref_crbm_cd(ker, bv, bh, v0, lr, seed):
    """The reference's own crbm_cd_update with std::mt19937(seed) (oracle/_ref)."""
    lib = load("ref")
    ker = np.array(ker, np.float32, copy=True, order="C")
    bv = np.array(bv, np.float32, copy=True)
    bh = np.array(bh, np.float32, copy=True)
    v0 = np.ascontiguousarray(v0, np.float32)
    k, c, kh, kw = ker.shape
    B, _, h, w = v0.shape
    recon = lib.ref_crbm_cd(c, h, w, k, kh, kw, fptr(ker), fptr(bv), fptr(bh), fptr(v0), B, lr, seed)
    return recon, ker, bv, bh


def crbm_init(c: int, h: int, w: int, k: int, kh: int, kw: int, seed: int, which: str = "oracle") -> np.ndarray:
    lib = load(which)
    ker = np.zeros((k, c, kh, kw), np.float32)
    if which == "oracle":
        lib.orc_crbm_init(c, k, kh, kw, seed, fptr(ker))
    else:
        lib.ref_crbm_init(c, h, w, k, kh, kw, seed, fptr(ker))
    return ker


def uniform_f32(seed: int, n: int, lo: float = 0.0, hi: float = 1.0) -> np.ndarray:
    out = np.zeros(n, np.float32)
    load().orc_uniform_f32(seed, lo, hi, n, fptr(out))
    return out


def canonical_f64(seed: int, n: int) -> np.ndarray:
    """std::generate_canonical<double,53>(std::mt19937(seed)) stream: the uniforms behind
    std::bernoulli_distribution (libstdc++ random.h:3741-3749)."""
    out = np.zeros(n, np.float64)
    load().orc_canonical_f64(seed, n, dptr(out))
    return out


def bernoulli_f32(seed: int, p: float, n: int) -> np.ndarray:
    out = np.zeros(n, np.float32)
    load().orc_bernoulli_f32(seed, p, n, fptr(out))
    return out


def uniform_int(seed: int, lo: int, hi: int, n: int) -> np.ndarray:
    out = np.zeros(n, np.int32)
    load().orc_uniform_int(seed, lo, hi, n, iptr(out))
    return out


def conv_forward(x, ker, bias, pad=0):
    lib = load()
    x = np.ascontiguousarray(x, np.float32)
    ker = np.ascontiguousarray(ker, np.float32)
    n, c, h, w = x.shape
    k, _, kh, kw = ker.shape
    y = np.zeros((n, k, h + 2 * pad - kh + 1, w + 2 * pad - kw + 1), np.float32)
    b = np.ascontiguousarray(bias, np.float32)
    lib.orc_conv_forward(fptr(x), n, c, h, w, fptr(ker), fptr(b), k, kh, kw, pad, fptr(y))
    return y


def conv_backward(x, ker, dy, pad=0):
    lib = load()
    x = np.ascontiguousarray(x, np.float32)
    ker = np.ascontiguousarray(ker, np.float32)
    dy = np.ascontiguousarray(dy, np.float32)
    n, c, h, w = x.shape
    k, _, kh, kw = ker.shape
    dx = np.zeros_like(x)
    gk = np.zeros_like(ker)
    gb = np.zeros(k, np.float32)
    lib.orc_conv_backward(fptr(x), n, c, h, w, fptr(ker), k, kh, kw, pad, fptr(dy), fptr(dx), fptr(gk), fptr(gb))
    return dx, gk, gb
