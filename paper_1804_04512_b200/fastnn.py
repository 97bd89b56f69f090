"""Host-side mirror of the reference's hot-path API (fastnn, /root/reference/proj/include/fastnn).

Same names, argument meaning and error types as the reference, backed by the B200 C ABI
(include/b200nn.h). Tensors are numpy arrays in fastnn's logical layout (NCHW / (out, in) /
(k, c, kh, kw)); parameters stay resident on the GPU between steps.

    spec = NetworkSpec(input=[784], layers=[LayerDesc.dense(784, 500), LayerDesc.sigmoid(), ...])
    net = build_network(spec)                      # network.hpp:284
    loss = train_minibatch(net, x, y_onehot)       # network.hpp:463
    probs = forward_batch(net, x)                  # network.hpp:402
    acc = evaluate(net, images, labels)            # network.hpp:474
    report = fit(net, images, labels, epochs)      # network.hpp:488
    rbm = Rbm(500, 784); rbm.init(seed)            # energy.hpp:16-32
    recon = cd_k_update(rbm, v0, 1, lr, uniforms)  # energy.hpp:131
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from ._lib import (BoundsError, ConsistencyError, CudaError, DataError, DataMissingError, Error,  # noqa: F401
                   FormatError, LabelError, LengthError, NcclError, ParamError, ShapeError, SpecError)

DENSE, CONV, MAXPOOL, SIGMOID, RELU, SOFTMAX, DROPOUT, BATCHNORM, FLATTEN = range(9)
TF32X3, TF32 = 0, 1
VALUE, GRAD, VELOCITY, OPT_STATE1, OPT_STATE2 = 0, 1, 2, 3, 4  # OPT_STATE1/2: acc/acc_update or adam m/v
SGD_MOMENTUM, ADAGRAD, ADADELTA, ADAM = 0, 1, 2, 3  # OptimizerKind (optim.hpp:11)


def _f(a: np.ndarray):
    return a.ctypes.data_as(C.POINTER(C.c_float))


def _d(a: np.ndarray):
    return a.ctypes.data_as(C.POINTER(C.c_double))


def _i(a: np.ndarray):
    return a.ctypes.data_as(C.POINTER(C.c_int))


@dataclass
class LayerDesc:
    """fastnn::LayerDesc (network.hpp:194-223) plus conv `pad`."""
    kind: int = DENSE
    in_: int = 0
    out: int = 0
    k: int = 0
    kh: int = 0
    kw: int = 0
    pad: int = 0
    p: float = 0.0

    @staticmethod
    def dense(i: int, o: int) -> "LayerDesc":
        return LayerDesc(DENSE, in_=i, out=o)

    @staticmethod
    def conv(k: int, kh: int, kw: int, pad: int = 0) -> "LayerDesc":
        return LayerDesc(CONV, k=k, kh=kh, kw=kw, pad=pad)

    @staticmethod
    def maxpool() -> "LayerDesc":
        return LayerDesc(MAXPOOL)

    @staticmethod
    def sigmoid() -> "LayerDesc":
        return LayerDesc(SIGMOID)

    @staticmethod
    def relu() -> "LayerDesc":
        return LayerDesc(RELU)

    @staticmethod
    def softmax() -> "LayerDesc":
        return LayerDesc(SOFTMAX)

    @staticmethod
    def flatten() -> "LayerDesc":
        return LayerDesc(FLATTEN)

    @staticmethod
    def dropout(p: float) -> "LayerDesc":
        return LayerDesc(DROPOUT, p=p)

    @staticmethod
    def from_dict(d: dict) -> "LayerDesc":
        return LayerDesc(d["kind"], in_=d.get("in", 0), out=d.get("out", 0), k=d.get("k", 0), kh=d.get("kh", 0),
                         kw=d.get("kw", 0), pad=d.get("pad", 0), p=d.get("p", 0.0))


@dataclass
class NetworkSpec:
    """fastnn::NetworkSpec (network.hpp:225-234)."""
    input: list = field(default_factory=list)
    layers: list = field(default_factory=list)
    optimizer: int = 0
    lr: float = 0.1
    momentum: float = 0.9
    weight_decay: float = 0.0
    batch_size: int = 100
    seed: int = 42

    @staticmethod
    def from_dict(d: dict) -> "NetworkSpec":
        return NetworkSpec(input=list(d["input"]), layers=[LayerDesc.from_dict(x) for x in d["layers"]],
                           lr=d.get("lr", 0.1), momentum=d.get("momentum", 0.9),
                           weight_decay=d.get("weight_decay", 0.0), batch_size=d.get("batch_size", 100),
                           seed=d.get("seed", 42), optimizer=d.get("optimizer", 0))


class Network:
    """Device-resident fastnn::Network. Build with build_network()."""

    def __init__(self, spec: NetworkSpec, device: int = 0, precision: int = TF32X3):
        if isinstance(spec, dict):
            spec = NetworkSpec.from_dict(spec)
        self.spec = spec
        arr = (_lib.LayerDescC * max(len(spec.layers), 1))()
        for i, d in enumerate(spec.layers):
            arr[i].kind, arr[i].in_, arr[i].out = d.kind, d.in_, d.out
            arr[i].k, arr[i].kh, arr[i].kw, arr[i].pad, arr[i].p = d.k, d.kh, d.kw, d.pad, d.p
        cs = _lib.NetworkSpecC()
        cs.input_rank = len(spec.input)
        for i, e in enumerate(spec.input[:3]):
            cs.input[i] = e
        cs.layers = arr
        cs.n_layers = len(spec.layers)
        cs.optimizer = spec.optimizer
        cs.lr, cs.momentum, cs.weight_decay = spec.lr, spec.momentum, spec.weight_decay
        cs.batch_size = spec.batch_size
        cs.seed = spec.seed
        h = C.c_void_p()
        _lib.call("b2n_build_network", C.byref(cs), device, precision, C.byref(h))
        self._h = h
        self.input = list(spec.input)
        dense = [d for d in spec.layers if d.kind == DENSE]
        self.classes = dense[-1].out if dense else 0
        self.batch_size = spec.batch_size

    def __del__(self):
        h = getattr(self, "_h", None)
        if h:
            _lib.load().b2n_net_destroy(h)
            self._h = None

    @property
    def handle(self):
        return self._h

    # ---- fastnn::Network::trainable() surface
    def num_params(self) -> int:
        n = C.c_int()
        _lib.call("b2n_net_num_params", self._h, C.byref(n))
        return n.value

    def param_shape(self, idx: int) -> tuple:
        r = C.c_int()
        dims = (C.c_longlong * 4)()
        _lib.call("b2n_net_param_shape", self._h, idx, C.byref(r), dims)
        return tuple(dims[i] for i in range(r.value))

    def get_param(self, idx: int, which: int = VALUE) -> np.ndarray:
        out = np.zeros(self.param_shape(idx), np.float32)
        _lib.call("b2n_net_get_param", self._h, idx, which, _f(out))
        return out

    def set_param(self, idx: int, values, which: int = VALUE) -> None:
        v = np.ascontiguousarray(values, np.float32).reshape(self.param_shape(idx))
        _lib.call("b2n_net_set_param", self._h, idx, which, _f(v))

    def params(self, which: int = VALUE) -> list:
        return [self.get_param(i, which) for i in range(self.num_params())]

    def set_hparams(self, lr: float, momentum: float, weight_decay: float = 0.0) -> None:
        _lib.call("b2n_net_set_hparams", self._h, lr, momentum, weight_decay)

    # ---- inspection
    def layer_output(self, layer: int, batch: int, shape) -> tuple[np.ndarray, np.ndarray]:
        """(output, pool codes) of fused layer `layer` from the last forward, NCHW per row."""
        out = np.zeros([batch] + list(shape), np.float32)
        codes = np.zeros(out.shape, np.uint8)
        _lib.call("b2n_net_layer_output", self._h, layer, batch, _f(out), codes.ctypes.data_as(C.POINTER(C.c_ubyte)))
        return out, codes

    # ---- data-parallel pieces
    def forward_backward(self, x, labels, batch_global: int | None = None) -> float:
        x = np.ascontiguousarray(x, np.float32)
        labels = np.ascontiguousarray(labels, np.int32)
        out = C.c_double()
        _lib.call("b2n_net_forward_backward", self._h, _f(x), _i(labels), labels.shape[0],
                  batch_global or labels.shape[0], C.byref(out))
        return out.value

    def apply_update(self) -> None:
        _lib.call("b2n_net_apply_update", self._h)

    def dp_init(self, nccl_id: bytes, rank: int, world: int) -> None:
        _lib.call("b2n_net_dp_init", self._h, nccl_id, rank, world)

    # ---- device-resident stepping (bench)
    def stage(self, x, labels) -> None:
        x = np.ascontiguousarray(x, np.float32)
        labels = np.ascontiguousarray(labels, np.int32)
        _lib.call("b2n_net_stage", self._h, _f(x), _i(labels), labels.shape[0])

    def run_staged(self, steps: int, batch_global: int = 0) -> None:
        _lib.call("b2n_net_run_staged", self._h, steps, batch_global)

    def train_stream(self, x, labels, batch: int) -> np.ndarray:
        """train_minibatch over consecutive host batches (rows [i*batch, (i+1)*batch) per step),
        step i+1's host->device copy overlapped with step i; returns every step's loss."""
        xb = _flat_batch(self, x)
        lab = np.ascontiguousarray(labels, np.int32)
        if xb.shape[0] % batch or lab.shape[0] != xb.shape[0]:
            raise ShapeError("train_stream: x / labels must hold steps * batch rows")
        out = np.zeros(xb.shape[0] // batch, np.float64)
        _lib.call("b2n_net_train_stream", self._h, _f(xb), _i(lab), xb.shape[0] // batch, batch, _d(out))
        return out

    def loss(self) -> float:
        out = C.c_double()
        _lib.call("b2n_net_loss", self._h, C.byref(out))
        return out.value

    def stream_handle(self) -> int:
        s = C.c_void_p()
        _lib.call("b2n_net_stream", self._h, C.byref(s))
        return s.value or 0

    def kernels_per_step(self, batch: int) -> int:
        n = C.c_int()
        _lib.call("b2n_net_kernels_per_step", self._h, batch, C.byref(n))
        return n.value


def build_network(spec, device: int = 0, precision: int = TF32X3) -> Network:
    """fastnn::build_network (network.hpp:284-375)."""
    return Network(spec, device, precision)


def _flat_batch(net: Network, x) -> np.ndarray:
    x = np.ascontiguousarray(x, np.float32)
    per = int(np.prod(net.input))
    if x.ndim < 2 or int(np.prod(x.shape[1:])) != per:  # network.hpp:380-392 ingest
        raise ShapeError("network input expects (batch, " + ", ".join(str(e) for e in net.input) + ")")
    return x.reshape(x.shape[0], per)


def train_minibatch(net: Network, x, y_onehot) -> float:
    """fastnn::train_minibatch (network.hpp:463-472); y is one-hot (batch, classes)."""
    xb = _flat_batch(net, x)
    y = np.ascontiguousarray(y_onehot, np.float32)
    if y.ndim != 2 or y.shape[0] != xb.shape[0] or y.shape[1] != net.classes:
        raise ShapeError("softmax_cross_entropy: predictions and labels must both be (batch, classes)")
    out = C.c_double()
    _lib.call("b2n_train_minibatch", net.handle, _f(xb), _f(y), xb.shape[0], C.byref(out))
    return out.value


def train_minibatch_labels(net: Network, x, labels) -> float:
    xb = _flat_batch(net, x)
    lab = np.ascontiguousarray(labels, np.int32)
    out = C.c_double()
    _lib.call("b2n_train_minibatch_labels", net.handle, _f(xb), _i(lab), xb.shape[0], C.byref(out))
    return out.value


def forward_batch(net: Network, x, return_argmax: bool = False):
    """fastnn::forward_batch (network.hpp:402); optional argmax_row ids (network.hpp:66-72)."""
    xb = _flat_batch(net, x)
    probs = np.zeros((xb.shape[0], net.classes), np.float32)
    am = np.zeros(xb.shape[0], np.int32)
    _lib.call("b2n_forward_batch", net.handle, _f(xb), xb.shape[0], _f(probs), _i(am))
    return (probs, am) if return_argmax else probs


def _dataset(net: Network, images, labels):
    x = _flat_batch(net, images)
    lab = np.ascontiguousarray(labels, np.int32)
    if lab.ndim != 1 or lab.shape[0] != x.shape[0]:
        raise ShapeError("dataset: need one label per image")
    if x.shape[0] == 0:
        raise DataError("empty dataset")
    return x, lab


def evaluate(net: Network, images, labels) -> float:
    """fastnn::evaluate (network.hpp:474-484): forward_batch in net.batch_size chunks over the
    device-resident dataset, first-max argmax accuracy counted on the device."""
    x, lab = _dataset(net, images, labels)
    out = C.c_double()
    _lib.call("b2n_net_evaluate", net.handle, _f(x), _i(lab), x.shape[0], C.byref(out))
    return out.value


@dataclass
class EpochStats:
    """fastnn::EpochStats (network.hpp:255-259)"""
    loss: float = 0.0
    accuracy: float = 0.0
    seconds: float = 0.0


@dataclass
class TrainReport:
    """fastnn::TrainReport (network.hpp:261-265)"""
    epochs: list = field(default_factory=list)
    test_accuracy: float = -1.0
    total_batches: int = 0


def fit(net: Network, images, labels, epochs: int, test=None) -> TrainReport:
    """fastnn::fit (network.hpp:488-511): `epochs` passes in BatchIterator order (net.seed,
    reshuffled with seed + epoch), the dataset resident in HBM and each batch gathered on the
    device; per-epoch mean loss, train accuracy and batch-loop seconds. `test` = (images, labels)."""
    x, lab = _dataset(net, images, labels)
    if epochs < 1:
        raise ParamError("fit: epochs must be >= 1")
    loss = np.zeros(epochs)
    acc = np.zeros(epochs)
    sec = np.zeros(epochs)
    _lib.call("b2n_net_fit", net.handle, _f(x), _i(lab), x.shape[0], epochs, _d(loss), _d(acc), _d(sec))
    rep = TrainReport([EpochStats(float(a), float(b), float(c)) for a, b, c in zip(loss, acc, sec)])
    rep.total_batches = epochs * -(-x.shape[0] // net.batch_size)
    if test is not None:
        rep.test_accuracy = evaluate(net, *test)
    return rep


def save_network(net: Network, path: str, with_state: bool = False) -> None:
    """fastnn::save_network (network.hpp:552-573): the reference's FNN1 bytes; with_state also
    writes `<path>.state` (momentum velocities + hyper-parameters) for an exact resume."""
    _lib.call("b2n_save_network", net.handle, str(path).encode(), int(with_state))


def load_network(net: Network, path: str, with_state: bool = False) -> None:
    """fastnn::load_network (network.hpp:575-607), same checks and error types."""
    _lib.call("b2n_load_network", net.handle, str(path).encode(), int(with_state))


def batch_order(n: int, seed: int, epoch: int = 0) -> np.ndarray:
    """BatchIterator's sample order (data.hpp:224-238) for epoch `epoch` of fit()."""
    out = np.zeros(n, np.int64)
    _lib.call("b2n_batch_order", n, seed, epoch, out.ctypes.data_as(C.POINTER(C.c_longlong)))
    return out


class Rbm:
    """fastnn::Rbm (energy.hpp:16-32), binary units, resident on the GPU."""

    def __init__(self, hidden: int, visible: int, device: int = 0, precision: int = TF32X3):
        h = C.c_void_p()
        _lib.call("b2n_rbm_create", hidden, visible, device, precision, C.byref(h))
        self._h = h
        self.hidden, self.visible = hidden, visible

    def __del__(self):
        h = getattr(self, "_h", None)
        if h:
            _lib.load().b2n_rbm_destroy(h)
            self._h = None

    @property
    def handle(self):
        return self._h

    def init(self, seed: int) -> None:
        _lib.call("b2n_rbm_init", self._h, seed)

    def set(self, w, bv, bh) -> None:
        w = np.ascontiguousarray(w, np.float32)
        bv = np.ascontiguousarray(bv, np.float32)
        bh = np.ascontiguousarray(bh, np.float32)
        if w.shape != (self.hidden, self.visible) or bv.shape != (self.visible,) or bh.shape != (self.hidden,):
            raise ShapeError("rbm parameter shapes")
        _lib.call("b2n_rbm_set", self._h, _f(w), _f(bv), _f(bh))

    def get(self):
        w = np.zeros((self.hidden, self.visible), np.float32)
        bv = np.zeros(self.visible, np.float32)
        bh = np.zeros(self.hidden, np.float32)
        _lib.call("b2n_rbm_get", self._h, _f(w), _f(bv), _f(bh))
        return w, bv, bh

    def kernels_per_step(self) -> int:
        n = C.c_int()
        _lib.call("b2n_rbm_kernels_per_step", self._h, C.byref(n))
        return n.value

    def last_states(self, batch: int):
        h0 = np.zeros((batch, self.hidden), np.float32)
        hs = np.zeros_like(h0)
        v1 = np.zeros((batch, self.visible), np.float32)
        h1 = np.zeros_like(h0)
        _lib.call("b2n_rbm_last_states", self._h, _f(h0), _f(hs), _f(v1), _f(h1))
        return h0, hs, v1, h1

    def set_rng(self, rng: "Mt19937") -> None:
        """load the caller's generator into the device generator (steps given no uniforms draw from it)"""
        st = rng.state()
        _lib.call("b2n_rbm_set_rng", self._h, st.ctypes.data_as(C.POINTER(C.c_uint)))

    def get_rng(self, rng: "Mt19937") -> None:
        """advance the caller's generator to the device generator's state"""
        st = np.zeros(625, np.uint32)
        _lib.call("b2n_rbm_get_rng", self._h, st.ctypes.data_as(C.POINTER(C.c_uint)))
        rng.set_state(st)

    def stage(self, v0, uniforms) -> None:
        """stage v0 and the uniforms (an array, or None: the device generator draws them)"""
        v0 = np.ascontiguousarray(v0, np.float32)
        if uniforms is None:
            _lib.call("b2n_rbm_stage", self._h, _f(v0), None, v0.shape[0])
            return
        u = np.ascontiguousarray(uniforms, np.float64)
        _lib.call("b2n_rbm_stage", self._h, _f(v0), _d(u), v0.shape[0])

    def run_staged(self, steps: int, lr: float, batch_global: int = 0) -> None:
        _lib.call("b2n_rbm_run_staged", self._h, steps, lr, batch_global)

    def recon(self) -> float:
        out = C.c_double()
        _lib.call("b2n_rbm_recon", self._h, C.byref(out))
        return out.value

    # ---- data parallelism driven by the caller (b2n_rbm_set_grad_only)
    def set_grad_only(self, on: bool) -> None:
        _lib.call("b2n_rbm_set_grad_only", self._h, 1 if on else 0)

    def get_grad(self):
        w = np.zeros((self.hidden, self.visible), np.float32)
        bv = np.zeros(self.visible, np.float32)
        bh = np.zeros(self.hidden, np.float32)
        _lib.call("b2n_rbm_get_grad", self._h, _f(w), _f(bv), _f(bh))
        return w, bv, bh

    def set_grad(self, w, bv, bh) -> None:
        w = np.ascontiguousarray(w, np.float32)
        bv = np.ascontiguousarray(bv, np.float32)
        bh = np.ascontiguousarray(bh, np.float32)
        _lib.call("b2n_rbm_set_grad", self._h, _f(w), _f(bv), _f(bh))

    def apply_update(self, lr: float, batch_global: int) -> None:
        _lib.call("b2n_rbm_apply_update", self._h, lr, batch_global)

    def train_stream(self, v0, uniforms, batch: int, lr: float) -> np.ndarray:
        """CD-1 over consecutive host batches (rows [i*batch, (i+1)*batch) of v0 / uniforms per
        step), copies of step i+1 overlapped with step i; returns every step's recon error."""
        v0 = np.ascontiguousarray(v0, np.float32)
        if v0.ndim != 2 or v0.shape[1] != self.visible or v0.shape[0] % batch:
            raise ShapeError("train_stream: v0 must be (steps * batch, visible)")
        steps = v0.shape[0] // batch
        out = np.zeros(steps, np.float64)
        if isinstance(uniforms, Mt19937):  # each step's draws generated on the device ahead of it
            self.set_rng(uniforms)
            _lib.call("b2n_rbm_train_stream", self._h, _f(v0), None, steps, batch, lr, _d(out))
            self.get_rng(uniforms)
            return out
        u = np.ascontiguousarray(uniforms, np.float64)
        if u.size < steps * batch * self.hidden:
            raise ShapeError("train_stream: need steps * batch * hidden uniforms")
        _lib.call("b2n_rbm_train_stream", self._h, _f(v0), _d(u), steps, batch, lr, _d(out))
        return out

    def train_stream_ptr(self, v0_ptr: int, u_ptr: int, steps: int, batch: int, lr: float) -> np.ndarray:
        """train_stream over device-resident batches: v0 (steps*batch x visible f32) and uniforms
        (steps*batch x hidden f64) at raw device addresses (e.g. torch tensors' data_ptr())"""
        out = np.zeros(steps, np.float64)
        _lib.call("b2n_rbm_train_stream", self._h, C.cast(C.c_void_p(v0_ptr), C.POINTER(C.c_float)), C.cast(C.c_void_p(u_ptr), C.POINTER(C.c_double)),
                  steps, batch, lr, _d(out))
        return out

    def stream_handle(self) -> int:
        s = C.c_void_p()
        _lib.call("b2n_rbm_stream", self._h, C.byref(s))
        return s.value or 0

    def dp_init(self, nccl_id: bytes, rank: int, world: int) -> None:
        _lib.call("b2n_rbm_dp_init", self._h, nccl_id, rank, world)


def cd_k_update(rbm: Rbm, v0, k: int, lr: float, uniforms, batch_global: int | None = None) -> float:
    """fastnn::cd_k_update (energy.hpp:131-171) with the Bernoulli uniforms supplied
    (k * batch * hidden generate_canonical<double,53> draws, the stream std::bernoulli_distribution
    consumes from the reference's std::mt19937)."""
    if k < 1:
        raise ParamError(f"cd_k_update: k must be >= 1, got {k}")
    v0 = np.ascontiguousarray(v0, np.float32)
    if v0.ndim != 2:
        raise ShapeError("cd_k_update: expected a rank-2 tensor")
    if v0.shape[1] != rbm.visible:
        raise ShapeError("cd_k_update: visible extent mismatch")
    out = C.c_double()
    if isinstance(uniforms, Mt19937):  # the draws on the device from the caller's generator
        rbm.set_rng(uniforms)
        _lib.call("b2n_cd_k_update", rbm.handle, _f(v0), v0.shape[0], k, lr, None, batch_global or v0.shape[0],
                  C.byref(out))
        rbm.get_rng(uniforms)
        return out.value
    u = np.ascontiguousarray(uniforms, np.float64).ravel()
    if u.size < k * v0.shape[0] * rbm.hidden:
        raise ShapeError("cd_k_update: need k * batch * hidden uniforms")
    _lib.call("b2n_cd_k_update", rbm.handle, _f(v0), v0.shape[0], k, lr, _d(u), batch_global or v0.shape[0],
              C.byref(out))
    return out.value


class Crbm:
    """fastnn::Crbm (energy.hpp:245-262), binary units, non-pooled, resident on the GPU.
    kernels (k, c_in, kh, kw), bv (c_in), bh (k); visible batches (n, c_in, h, w)."""

    def __init__(self, c_in: int, h: int, w: int, k: int, kh: int, kw: int, device: int = 0,
                 precision: int = TF32X3):
        hd = C.c_void_p()
        _lib.call("b2n_crbm_create", c_in, h, w, k, kh, kw, device, precision, C.byref(hd))
        self._h = hd
        self.c_in, self.h, self.w, self.k, self.kh, self.kw = c_in, h, w, k, kh, kw
        self.oh, self.ow = h - kh + 1, w - kw + 1

    def __del__(self):
        h = getattr(self, "_h", None)
        if h:
            _lib.load().b2n_crbm_destroy(h)
            self._h = None

    @property
    def handle(self):
        return self._h

    @property
    def kernel_shape(self):
        return (self.k, self.c_in, self.kh, self.kw)

    def init(self, seed: int) -> None:
        _lib.call("b2n_crbm_init", self._h, seed)

    def set(self, kernels, bv, bh) -> None:
        kernels = np.ascontiguousarray(kernels, np.float32)
        bv = np.ascontiguousarray(bv, np.float32)
        bh = np.ascontiguousarray(bh, np.float32)
        if kernels.shape != self.kernel_shape or bv.shape != (self.c_in,) or bh.shape != (self.k,):
            raise ShapeError("crbm parameter shapes")
        _lib.call("b2n_crbm_set", self._h, _f(kernels), _f(bv), _f(bh))

    def get(self):
        ker = np.zeros(self.kernel_shape, np.float32)
        bv = np.zeros(self.c_in, np.float32)
        bh = np.zeros(self.k, np.float32)
        _lib.call("b2n_crbm_get", self._h, _f(ker), _f(bv), _f(bh))
        return ker, bv, bh

    def kernels_per_step(self) -> int:
        n = C.c_int()
        _lib.call("b2n_crbm_kernels_per_step", self._h, C.byref(n))
        return n.value

    def dp_init(self, nccl_id: bytes, rank: int, world: int) -> None:
        _lib.call("b2n_crbm_dp_init", self._h, nccl_id, rank, world)

    def keep_states(self, on: bool = True) -> None:
        """write every step's chain states to HBM so last_states() can read them back"""
        _lib.call("b2n_crbm_keep_states", self._h, int(on))

    def last_states(self, batch: int):
        h0 = np.zeros((batch, self.k, self.oh, self.ow), np.float32)
        hs, h1 = np.zeros_like(h0), np.zeros_like(h0)
        v1 = np.zeros((batch, self.c_in, self.h, self.w), np.float32)
        _lib.call("b2n_crbm_last_states", self._h, _f(h0), _f(hs), _f(v1), _f(h1))
        return h0, hs, v1, h1

    def set_rng(self, rng: "Mt19937") -> None:
        st = rng.state()
        _lib.call("b2n_crbm_set_rng", self._h, st.ctypes.data_as(C.POINTER(C.c_uint)))

    def get_rng(self, rng: "Mt19937") -> None:
        st = np.zeros(625, np.uint32)
        _lib.call("b2n_crbm_get_rng", self._h, st.ctypes.data_as(C.POINTER(C.c_uint)))
        rng.set_state(st)

    def train_stream(self, v0, uniforms, batch: int, lr: float) -> np.ndarray:
        """crbm_cd_update over consecutive host batches of v0 (steps*batch images); uniforms = an array
        (steps*batch*k*oh*ow) or an Mt19937 (the draws generated on the device, rng advanced);
        returns every step's reconstruction error"""
        v0 = np.ascontiguousarray(v0, np.float32)
        if v0.ndim != 4 or v0.shape[1:] != (self.c_in, self.h, self.w) or v0.shape[0] % batch:
            raise ShapeError("train_stream: v0 must be (steps * batch, c_in, h, w)")
        steps = v0.shape[0] // batch
        out = np.zeros(steps, np.float64)
        if isinstance(uniforms, Mt19937):
            self.set_rng(uniforms)
            _lib.call("b2n_crbm_train_stream", self._h, _f(v0), None, steps, batch, lr, _d(out))
            self.get_rng(uniforms)
            return out
        u = np.ascontiguousarray(uniforms, np.float64)
        if u.size < steps * batch * self.k * self.oh * self.ow:
            raise ShapeError("train_stream: need steps * batch * k * oh * ow uniforms")
        _lib.call("b2n_crbm_train_stream", self._h, _f(v0), _d(u), steps, batch, lr, _d(out))
        return out

    def stage(self, v0, uniforms) -> None:
        """stage v0 and the uniforms (an array, or None: the device generator draws them)"""
        v0 = np.ascontiguousarray(v0, np.float32)
        if uniforms is None:
            if v0.ndim != 4 or v0.shape[1:] != (self.c_in, self.h, self.w):
                raise ShapeError("crbm stage: visible batch does not match the model")
            _lib.call("b2n_crbm_stage", self._h, _f(v0), None, v0.shape[0])
            return
        u = np.ascontiguousarray(uniforms, np.float64)
        if v0.ndim != 4 or v0.shape[1:] != (self.c_in, self.h, self.w) or u.size < v0.shape[0] * self.k * self.oh * self.ow:
            raise ShapeError("crbm stage: visible batch / uniforms do not match the model")
        _lib.call("b2n_crbm_stage", self._h, _f(v0), _d(u), v0.shape[0])

    def run_staged(self, steps: int, lr: float, batch_global: int = 0) -> None:
        _lib.call("b2n_crbm_run_staged", self._h, steps, lr, batch_global)

    def recon(self) -> float:
        out = C.c_double()
        _lib.call("b2n_crbm_recon", self._h, C.byref(out))
        return out.value

    def stream_handle(self) -> int:
        s = C.c_void_p()
        _lib.call("b2n_crbm_stream", self._h, C.byref(s))
        return s.value or 0


def crbm_cd_update(m: Crbm, v0, lr: float, uniforms, batch_global: int | None = None) -> float:
    """fastnn::crbm_cd_update (energy.hpp:333-376) with the Bernoulli uniforms supplied
    (batch * k * oh * ow generate_canonical<double,53> draws in NCHW order, the stream
    unit_sample_inplace's std::bernoulli_distribution consumes). Returns the reconstruction error
    per image."""
    v0 = np.ascontiguousarray(v0, np.float32)
    if v0.ndim != 4 or v0.shape[1] != m.c_in or v0.shape[2] != m.h or v0.shape[3] != m.w:
        raise ShapeError("crbm_cd_update: input does not match the model's visible shape")
    out = C.c_double()
    if isinstance(uniforms, Mt19937):  # the draws on the device from the caller's generator
        m.set_rng(uniforms)
        _lib.call("b2n_crbm_cd_update", m.handle, _f(v0), v0.shape[0], lr, None, batch_global or v0.shape[0],
                  C.byref(out))
        m.get_rng(uniforms)
        return out.value
    u = np.ascontiguousarray(uniforms, np.float64).ravel()
    if u.size < v0.shape[0] * m.k * m.oh * m.ow:
        raise ShapeError("crbm_cd_update: need batch * k * oh * ow uniforms")
    _lib.call("b2n_crbm_cd_update", m.handle, _f(v0), v0.shape[0], lr, _d(u), batch_global or v0.shape[0],
              C.byref(out))
    return out.value


class Mt19937:
    """A std::mt19937 stream (numpy's MT19937 with the legacy init_genrand seeding is the same
    generator) yielding std::generate_canonical<double,53> values: two 32-bit draws per double,
    (lo + hi * 2^32) / 2^64, clamped below 1 -- exactly what std::bernoulli_distribution consumes."""

    def __init__(self, seed: int):
        self._rs = np.random.RandomState(seed)
        self._st = None  # the libstdc++ state when it is newer than _rs (set by the device generator)

    @property
    def _rs(self):
        if self._st is not None:  # bring the host generator up to the state the device left
            self.__rs.set_state(("MT19937", self._st[:624].copy(), int(self._st[624]), 0, 0.0))
            self._st = None
        return self.__rs

    @_rs.setter
    def _rs(self, rs):
        self.__rs = rs
        self._st = None

    def state(self) -> np.ndarray:
        """the libstdc++ state (_M_x[624], _M_p) as 625 uint32 -- what the device generator takes"""
        if self._st is not None:
            return self._st.copy()
        _, key, pos, _, _ = self.__rs.get_state(legacy=True)
        return np.concatenate([np.asarray(key, np.uint32), np.asarray([pos], np.uint32)])

    def set_state(self, st) -> None:
        """(kept as the 625 words; numpy's generator is re-seeded from them only when the host draws
        next -- a loop of device-drawn steps never pays for the conversion)"""
        self._st = np.array(st, np.uint32).reshape(625)

    def canonical(self, n: int) -> np.ndarray:
        u = self._rs.randint(0, 2 ** 32, size=2 * n, dtype=np.uint64).reshape(n, 2).astype(np.float64)
        c = (u[:, 0] + u[:, 1] * 4294967296.0) / 18446744073709551616.0
        return np.where(c >= 1.0, np.nextafter(1.0, 0.0), c)


_UNIFORM_FN = C.CFUNCTYPE(None, C.c_void_p, C.POINTER(C.c_double), C.c_longlong)


@dataclass
class DbnReport:
    """fastnn::DbnReport (energy.hpp:199-201): recon[layer][epoch]"""
    recon: list = field(default_factory=list)


def dbn_pretrain(stack: list, data, epochs: int, lr: float, batch_size: int, rng: Mt19937,
                 host_draws: bool = False) -> DbnReport:
    """fastnn::dbn_pretrain (energy.hpp:208-240): greedy CD-1 over a stack of Rbm on one device,
    data resident in HBM, each layer's hidden means computed on the device for the next; the
    Bernoulli uniforms are drawn from `rng` in the reference's order (B x H per step) -- on the
    device (default; `rng` is advanced to match), or on the host through a callback."""
    data = np.ascontiguousarray(data, np.float32)
    if data.ndim != 2:
        raise ShapeError("dbn_pretrain: data must be (rows, visible)")
    arr = (C.c_void_p * max(len(stack), 1))(*[r.handle.value if hasattr(r.handle, "value") else r.handle
                                               for r in stack])

    if not host_draws:
        st = rng.state()
        rec = np.zeros(max(len(stack) * epochs, 1))
        _lib.call("b2n_dbn_pretrain", arr, len(stack), _f(data), data.shape[0], epochs, lr, batch_size, None,
                  st.ctypes.data_as(C.c_void_p), _d(rec))
        rng.set_state(st)
        return DbnReport([list(rec[l * epochs:(l + 1) * epochs]) for l in range(len(stack))])

    def fill(_ctx, out, count):
        np.ctypeslib.as_array(out, shape=(count,))[:] = rng.canonical(count)

    cb = _UNIFORM_FN(fill)
    rec = np.zeros(max(len(stack) * epochs, 1))
    _lib.call("b2n_dbn_pretrain", arr, len(stack), _f(data), data.shape[0], epochs, lr, batch_size,
              C.cast(cb, C.c_void_p), None, _d(rec))
    return DbnReport([list(rec[l * epochs:(l + 1) * epochs]) for l in range(len(stack))])


def mt19937_draw(rng: Mt19937, n: int, device: int = 0) -> np.ndarray:
    """the next n generate_canonical<double,53> draws of `rng`, generated on the GPU (rng advanced)"""
    st = rng.state()
    out = np.zeros(max(n, 1), np.float64)
    _lib.call("b2n_mt19937_draw", device, st.ctypes.data_as(C.POINTER(C.c_uint)), _d(out), n)
    rng.set_state(st)
    return out[:n]


# ---------------------------------------------------------------- the reference's op-level layer API
# (layers.hpp:124-320, network.hpp:410-437) on the GPU, bit-identical to fastnn's: host arrays in / out.
SIGMOID, RELU = 0, 1      # Activation (layers.hpp:276)
POOL_MAX, POOL_AVG = 0, 1  # PoolMode (layers.hpp:197)


class _ConvShapeC(C.Structure):
    _fields_ = [(n, C.c_longlong) for n in ("n", "c_in", "k", "kh", "kw", "h", "w", "pad")]


def _conv_shape(x, kernels, pad):
    n, c, h, w = x.shape
    k, c2, kh, kw = kernels.shape
    if c2 != c:
        raise ShapeError("conv: input channels do not match the kernels")
    return _ConvShapeC(n, c, k, kh, kw, h, w, pad)


def conv_forward(kernels, bias, x, pad: int = 0, device: int = 0) -> np.ndarray:
    """fastnn::conv_forward (layers.hpp:132): x (n, c_in, h, w), kernels (k, c_in, kh, kw), bias (k)"""
    x = np.ascontiguousarray(x, np.float32)
    kernels = np.ascontiguousarray(kernels, np.float32)
    bias = np.ascontiguousarray(bias, np.float32)
    if x.ndim != 4:
        raise ShapeError("conv_forward: expected a rank-4 input")
    s = _conv_shape(x, kernels, pad)
    y = np.zeros((s.n, s.k, s.h + 2 * pad - s.kh + 1, s.w + 2 * pad - s.kw + 1), np.float32)
    _lib.call("b2n_op_conv_forward", device, C.addressof(s), _f(x), _f(kernels), _f(bias), _f(y))
    return y


def conv_backward(kernels, x, dy, gk, gb, device: int = 0) -> np.ndarray:
    """fastnn::conv_backward (layers.hpp:152): returns dx; gk (k, c_in, kh, kw) and gb (k) are float32
    arrays that accumulate in place, as the layer's gradient tensors do"""
    x = np.ascontiguousarray(x, np.float32)
    dy = np.ascontiguousarray(dy, np.float32)
    kernels = np.ascontiguousarray(kernels, np.float32)
    if x.ndim != 4 or dy.ndim != 4:
        raise ShapeError("conv_backward: expected rank-4 tensors")
    if gk.dtype != np.float32 or gb.dtype != np.float32 or not gk.flags.c_contiguous or not gb.flags.c_contiguous:
        raise ParamError("conv_backward: gk / gb must be contiguous float32 arrays (updated in place)")
    s = _conv_shape(x, kernels, 0)
    if dy.shape != (s.n, s.k, s.h - s.kh + 1, s.w - s.kw + 1):
        raise ShapeError("conv_backward: dy does not match the forward output shape")
    dx = np.zeros_like(x)
    _lib.call("b2n_op_conv_backward", device, C.addressof(s), _f(x), _f(kernels), _f(dy), _f(gk), _f(gb), _f(dx))
    return dx


def pool_forward(mode: int, x, device: int = 0):
    """fastnn::pool_forward (layers.hpp:205): 2x2 windows over the last two axes; returns (y, argmax)
    (argmax None in avg mode)"""
    x = np.ascontiguousarray(x, np.float32)
    if x.ndim < 2:
        raise ShapeError("pool_forward: expected rank >= 2")
    h, w = x.shape[-2:]
    maps = int(np.prod(x.shape[:-2])) if x.ndim > 2 else 1
    oshape = x.shape[:-2] + (h // 2, w // 2)
    y = np.zeros(oshape, np.float32)
    a = np.zeros(oshape, np.float32) if mode == POOL_MAX else None
    _lib.call("b2n_op_pool_forward", device, mode, maps, h, w, _f(x), _f(y), _f(a) if a is not None else None)
    return y, a


def pool_backward(mode: int, dy, argmax=None, device: int = 0) -> np.ndarray:
    """fastnn::pool_backward (layers.hpp:240)"""
    dy = np.ascontiguousarray(dy, np.float32)
    if dy.ndim < 2:
        raise ShapeError("pool_backward: expected rank >= 2")
    if mode == POOL_MAX and (argmax is None or np.shape(argmax) != dy.shape):
        raise ShapeError("pool_backward: dy/argmax shape mismatch")
    oh, ow = dy.shape[-2:]
    maps = int(np.prod(dy.shape[:-2])) if dy.ndim > 2 else 1
    dx = np.zeros(dy.shape[:-2] + (2 * oh, 2 * ow), np.float32)
    a = np.ascontiguousarray(argmax, np.float32) if mode == POOL_MAX else None
    _lib.call("b2n_op_pool_backward", device, mode, maps, oh, ow, _f(dy), _f(a) if a is not None else None, _f(dx))
    return dx


def activation_apply(kind: int, x, device: int = 0) -> np.ndarray:
    """fastnn::activation_apply (layers.hpp:278)"""
    x = np.ascontiguousarray(x, np.float32)
    y = np.zeros_like(x)
    _lib.call("b2n_op_activation_apply", device, kind, x.size, _f(x), _f(y))
    return y


def activation_gradient(kind: int, y, dy, device: int = 0) -> np.ndarray:
    """fastnn::activation_gradient (layers.hpp:284), through the forward output y"""
    y = np.ascontiguousarray(y, np.float32)
    dy = np.ascontiguousarray(dy, np.float32)
    if y.shape != dy.shape:
        raise ShapeError("activation_gradient: shape mismatch")
    dx = np.zeros_like(y)
    _lib.call("b2n_op_activation_gradient", device, kind, y.size, _f(y), _f(dy), _f(dx))
    return dx


def softmax(x, device: int = 0) -> np.ndarray:
    """fastnn::softmax (layers.hpp:301)"""
    x = np.ascontiguousarray(x, np.float32)
    if x.ndim != 2:
        raise ShapeError(f"softmax: expected a rank-2 tensor, got rank {x.ndim}")
    y = np.zeros_like(x)
    _lib.call("b2n_op_softmax", device, x.shape[0], x.shape[1], _f(x), _f(y))
    return y


def softmax_cross_entropy(predictions, labels, device: int = 0):
    """fastnn::softmax_cross_entropy (network.hpp:410): returns (loss, dlogits)"""
    p = np.ascontiguousarray(predictions, np.float32)
    y = np.ascontiguousarray(labels, np.float32)
    if p.ndim != 2 or y.ndim != 2 or p.shape != y.shape:
        raise ShapeError("softmax_cross_entropy: predictions and labels must both be (batch, classes)")
    g = np.zeros_like(p)
    loss = C.c_double()
    _lib.call("b2n_op_softmax_cross_entropy", device, p.shape[0], p.shape[1], _f(p), _f(y), _f(g), C.byref(loss))
    return loss.value, g


def nccl_unique_id() -> bytes:
    buf = C.create_string_buffer(128)
    _lib.call("b2n_nccl_unique_id", buf)
    return buf.raw


# ---- op level on device tensors (torch CUDA tensors: plumbing only)
def gemm(a, b, transpose_a: bool = False, transpose_b: bool = False, precision: int = TF32X3):
    """fastnn::gemm (gemm.hpp:225-229) on CUDA tensors: C = op(A) . op(B)."""
    import torch
    M = a.shape[1] if transpose_a else a.shape[0]
    K = a.shape[0] if transpose_a else a.shape[1]
    kb = b.shape[1] if transpose_b else b.shape[0]
    N = b.shape[0] if transpose_b else b.shape[1]
    if K != kb:
        raise ShapeError(f"gemm inner extents disagree: {K} vs {kb}")
    c = torch.empty((M, N), dtype=torch.float32, device=a.device)
    stream = torch.cuda.current_stream(a.device).cuda_stream
    _lib.call("b2n_gemm", a.data_ptr(), a.stride(0), int(transpose_a), b.data_ptr(), b.stride(0), int(transpose_b),
              c.data_ptr(), c.stride(0), M, N, K, precision, stream)
    return c


def sgd_momentum_step(p, v, g, lr: float, momentum: float, weight_decay: float = 0.0) -> None:
    """fastnn::sgd_momentum_step (optim.hpp:69-80) on contiguous CUDA tensors, in place."""
    import torch
    stream = torch.cuda.current_stream(p.device).cuda_stream
    _lib.call("b2n_sgd_momentum_step", p.data_ptr(), v.data_ptr(), g.data_ptr(), p.numel(), lr, momentum,
              weight_decay, stream)
