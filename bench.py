#!/usr/bin/env python
"""Benchmark of the B200 data-parallel training step (BASELINE.json metric: train samples/s).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config rbm|mlp|mnist_cnn|cifar_cnn|imagenet_cnn]
                    [--impl ours|reference] [--precision tf32x3|tf32]

One JSON line on rank 0. The headline workload is BASELINE.json configs[1] (MNIST-shape RBM
784-500, CD-1, batch 100); the other configs are measured in the same run under "other_configs".
  value   : device-resident whole-job throughput (inputs staged in HBM once, each step one CUDA
            graph launch of the whole step; L2 flushed between timed steps; CUDA events on the
            library's stream; max over ranks).
  e2e     : the same metric through the public API call with pinned host buffers (H2D of the
            step's inputs and D2H of its loss / reconstruction inside the timed region).
  roofline: the dominant kernel's algorithmic bytes (or FLOPs) per launch / its event-timed
            duration vs MEASURED_PEAKS.json.
  cpu_baseline: the reference's own CPU step (oracle/_ref, compiled from /root/reference's headers)
            on this host's cores, bounded sample, rank 0 at N=1 only.
Multi-GPU: torchrun, one process per GPU, the global batch sharded (strong scaling), gradients
allreduced by NCCL inside the step graph.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

FLUSH_BYTES = 512 << 20  # > 126 MB L2, written between timed steps
NVML_REASONS = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap", 0x8: "hw_slowdown",
                0x10: "sync_boost", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown",
                0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting"}


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=200)
    p.add_argument("--warmup", type=int, default=20)
    p.add_argument("--config", default="rbm")
    p.add_argument("--impl", default="ours", choices=["ours", "reference"])
    p.add_argument("--precision", default="tf32x3", choices=["tf32x3", "tf32"])
    p.add_argument("--cpu-budget", type=float, default=12.0, help="seconds of reference CPU work to time")
    p.add_argument("--no-others", action="store_true", help="skip the other configs")
    p.add_argument("--profile-only", action="store_true", help="run the step loop only (for ncu)")
    return p.parse_args()


# ----------------------------------------------------------------------------- distributed
class Dist:
    def __init__(self):
        self.world = int(os.environ.get("WORLD_SIZE", "1"))
        self.rank = int(os.environ.get("RANK", "0"))
        self.local = int(os.environ.get("LOCAL_RANK", "0"))
        self.pg = None

    def init(self, backend="nccl"):
        import torch
        if self.world > 1:
            import torch.distributed as dist
            os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
            torch.cuda.set_device(self.local)
            dist.init_process_group(backend, rank=self.rank, world_size=self.world,
                                    device_id=torch.device("cuda", self.local))
            self.pg = dist

    def barrier(self):
        if self.pg:
            self.pg.barrier()

    def max(self, x: float) -> float:
        if not self.pg:
            return x
        import torch
        t = torch.tensor([x], dtype=torch.float64, device=f"cuda:{self.local}")
        self.pg.all_reduce(t, op=self.pg.ReduceOp.MAX)
        return float(t.item())

    def bcast_bytes(self, b: bytes | None) -> bytes:
        if not self.pg:
            return b
        obj = [b]
        self.pg.broadcast_object_list(obj, src=0)
        return obj[0]


# ----------------------------------------------------------------------------- clocks
class ClockSampler:
    def __init__(self, device_index: int):
        self.samples = []
        self.max_mhz = None
        self.reasons = 0
        self._stop = threading.Event()
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(device_index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self.nv = None

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                self.reasons |= self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
            except Exception:
                pass
            time.sleep(0.01)

    def __enter__(self):
        if self.nv:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self.nv:
            self.t.join()

    def summary(self):
        if not self.nv:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvml unavailable"]}
        reasons = [n for b, n in NVML_REASONS.items() if self.reasons & b and n != "gpu_idle"]
        return {"sm_mhz": statistics.median(self.samples) if self.samples else None, "sm_max_mhz": self.max_mhz,
                "reasons": reasons, "samples": len(self.samples)}


# ----------------------------------------------------------------------------- workloads
def pinned(shape, dtype):
    import torch
    tdt = {np.float32: torch.float32, np.float64: torch.float64, np.int32: torch.int32}[dtype]
    return torch.empty(shape, dtype=tdt, pin_memory=True).numpy()


class RbmWork:
    name = "rbm"

    def __init__(self, dist: Dist, precision: int, nccl_id):
        from oracle import oracle as O  # synthetic-input generators (std::mt19937 streams), not the measured path
        from paper_1804_04512_b200 import configs as CF, fastnn as F
        from paper_1804_04512_b200.dp import shard_bounds
        c = CF.RBM
        self.H, self.V, self.Bg, self.lr = c["hidden"], c["visible"], c["batch_size"], c["lr"]
        lo, hi = shard_bounds(self.Bg, dist.world, dist.rank)
        self.B = hi - lo
        v0 = O.bernoulli_f32(3, 0.5, self.Bg * self.V).reshape(self.Bg, self.V)[lo:hi]
        u = O.canonical_f64(5, self.Bg * self.H).reshape(self.Bg, self.H)[lo:hi]
        self.rbm = F.Rbm(self.H, self.V, device=dist.local, precision=precision)
        self.rbm.init(c["seed"])
        if dist.world > 1:
            self.rbm.dp_init(nccl_id, dist.rank, dist.world)
        self.rbm.stage(v0, u)
        self.v0_h = pinned(v0.shape, np.float32)
        self.v0_h[:] = v0
        self.u_h = pinned(u.shape, np.float64)
        self.u_h[:] = u
        self.F = F
        self.dist = dist
        self.config = {"workload": "mnist_rbm_cd1", "model": "RBM 784-500 binary, CD-1", "global_batch": self.Bg,
                       "local_batch": self.B, "parallelism": f"dp{dist.world}", "lr": self.lr,
                       "sampling": "std::mt19937 generate_canonical<double,53> stream (bit-exact Bernoulli): "
                                   "staged for `value`, generated on the device from the caller's generator "
                                   "inside the timed region for `e2e`"}
        self.h2d = self.B * self.V * 4  # e2e: v0 only -- the draws are generated on the device
        self.d2h = None

    def stream(self):
        return self.rbm.stream_handle()

    def step(self, n=1):
        self.rbm.run_staged(n, self.lr, self.Bg)

    def e2e_step(self):
        if getattr(self, "_gen1", None) is None:  # this rank's generator (device draws)
            self._gen1 = self.F.Mt19937(23 + self.dist.rank)
            self.rbm.set_rng(self._gen1)
        if self.dist.world > 1:  # data-parallel: stage the shard (H2D + device draws), one step, recon
            self.rbm.stage(self.v0_h, None)
            self.rbm.run_staged(1, self.lr, self.Bg)
            return self.rbm.recon()
        return self.F.cd_k_update(self.rbm, self.v0_h, 1, self.lr, self._gen1, self.Bg)

    def e2e_total(self, steps, warmup):
        """end to end through Rbm.train_stream (the loop of cd_k_update(rbm, v0_i, 1, lr, rng) calls
        over host batches): `steps` distinct pinned host batches (together larger than L2), every
        step's H2D inside the timed region (overlapped with the previous step), every step's
        Bernoulli draws generated from the caller's mt19937 inside it (on the device, ahead of the
        step), every step's recon read back. Returns the device time of the call (ms)."""
        if self.dist.world > 1:
            return None
        import torch
        from oracle import oracle as O  # synthetic-input generators (std::mt19937 streams), not the measured path
        n = steps * self.B
        if getattr(self, "_sv", None) is None or self._sv.shape[0] < n:
            self._sv = pinned((n, self.V), np.float32)
            self._sv[:] = O.bernoulli_f32(11, 0.5, n * self.V).reshape(n, self.V)
        # the Bernoulli draws: the reference's std::mt19937 stream generated on the device from the
        # caller's generator state (bit-exact; the state goes up once and comes back once per call)
        gen = self.F.Mt19937(13)
        self.rbm.train_stream(self._sv[:max(warmup, 1) * self.B], gen, self.B, self.lr)
        s = torch.cuda.ExternalStream(self.stream())
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        self.dist.barrier()
        torch.cuda.synchronize()
        e0.record(s)
        self.rbm.train_stream(self._sv[:n], gen, self.B, self.lr)
        e1.record(s)
        torch.cuda.synchronize()
        self.dist.barrier()
        return self.dist.max(e0.elapsed_time(e1))

    def value_total(self, steps, warmup, flush=None):
        """device throughput in steady state: `steps` consecutive CD-1 steps over distinct batches already
        resident in HBM (v0 + the reference's uniforms), L2 flushed before the timed call and no batch
        read twice inside it, through the same staging pipeline as e2e minus the PCIe. Returns the device
        time of the call (ms) on the library stream, or None when data-parallel."""
        if self.dist.world > 1:
            return None
        import torch
        from oracle import oracle as O  # synthetic-input generators (std::mt19937 streams), not the measured path
        n = steps * self.B
        dev = torch.device("cuda", self.dist.local)
        v = torch.from_numpy(O.bernoulli_f32(31, 0.5, n * self.V).reshape(n, self.V)).to(dev)
        u = torch.from_numpy(O.canonical_f64(37, n * self.H).reshape(n, self.H)).to(dev)
        w = max(warmup, 1)
        self.rbm.train_stream_ptr(v.data_ptr(), u.data_ptr(), w, self.B, self.lr)
        if flush is not None:  # nothing of the batches in L2 when the timed region starts (they were just written)
            flush.zero_()
        s = torch.cuda.ExternalStream(self.stream())
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record(s)
        self.rbm.train_stream_ptr(v.data_ptr(), u.data_ptr(), steps, self.B, self.lr)
        e1.record(s)
        torch.cuda.synchronize()
        self.value_bytes = v.nbytes + u.nbytes
        return e0.elapsed_time(e1)

    def kernels_per_step(self):
        return _kernels(self.F._lib, "b2n_rbm_kernels_per_step", self.rbm.handle)

    def stream_launches_per_step(self):  # train_stream: the fused step + stage_rows_kernel (tf32 lo of v0)
        return self.kernels_per_step() + 1

    def profile(self, steps):
        return _profile(self.F._lib, "b2n_rbm_profile", self.rbm.handle, steps, self.lr, self.Bg)

    def d2h_bytes(self):
        # fused step, single GPU, pinned inputs: the kernel reads v0 and the uniforms from host memory
        # and stores the finished recon (one double) into host-mapped memory; otherwise the per-
        # (tile, row) reconstruction partials are copied back (one tile per 64 visible columns)
        if self.kernels_per_step() == 1 and self.dist.world == 1:
            return 8
        return self.B * 8 * ((self.V + 63) // 64)


class CrbmWork:
    """CD-1 of the MNIST-shaped convolutional RBM (configs.CRBM), single GPU."""
    name = "crbm"

    def __init__(self, dist: Dist, precision: int, nccl_id):
        from oracle import oracle as O  # synthetic-input generators (std::mt19937 streams), not the measured path
        from paper_1804_04512_b200 import configs as CF, fastnn as F
        from paper_1804_04512_b200.dp import shard_bounds
        c = CF.CRBM
        self.Bg = c["batch_size"]
        lo, hi = shard_bounds(self.Bg, dist.world, dist.rank)
        self.B = hi - lo
        self.lr = c["lr"]
        shp = (c["c_in"], c["h"], c["w"])
        oh, ow = c["h"] - c["kh"] + 1, c["w"] - c["kw"] + 1
        v0 = O.bernoulli_f32(3, 0.5, self.Bg * int(np.prod(shp))).reshape((self.Bg,) + shp)[lo:hi]
        u = O.canonical_f64(5, self.Bg * c["k"] * oh * ow).reshape(self.Bg, -1)[lo:hi]
        self.m = F.Crbm(*shp, c["k"], c["kh"], c["kw"], device=dist.local, precision=precision)
        self.m.init(c["seed"])
        if dist.world > 1:
            self.m.dp_init(nccl_id, dist.rank, dist.world)
        self.m.stage(v0, u)
        self.dist = dist
        self.v0_h = pinned(v0.shape, np.float32)
        self.v0_h[:] = v0
        self.u_h = pinned(u.shape, np.float64)
        self.u_h[:] = u
        self.F = F
        self.config = {"workload": "mnist_crbm_cd1", "model": f"CRBM 1x28x28, {c['k']} kernels 5x5, binary, CD-1",
                       "global_batch": self.Bg, "local_batch": self.B, "parallelism": f"dp{dist.world}",
                       "lr": self.lr}
        self.h2d = v0.nbytes  # e2e: v0 only -- the draws are generated on the device

    def stream(self):
        return self.m.stream_handle()

    def step(self, n=1):
        self.m.run_staged(n, self.lr, self.Bg)

    def e2e_total(self, steps, warmup):
        """end to end through Crbm.train_stream (the loop of crbm_cd_update(m, v0_i, lr, rng) calls over
        host batches): `steps` distinct pinned host batches, each step's H2D and its 691,200 Bernoulli
        draws (generated on the device from the caller's mt19937, 16 steps in flight by jump-ahead)
        inside the timed region, every recon read back. Device time of the call (ms)."""
        if self.dist.world > 1:
            return None
        import torch
        from oracle import oracle as O  # synthetic-input generators (std::mt19937 streams), not the measured path
        n = steps * self.B
        shp = self.v0_h.shape[1:]
        if getattr(self, "_sv", None) is None or self._sv.shape[0] < n:
            self._sv = pinned((n,) + shp, np.float32)
            self._sv[:] = O.bernoulli_f32(11, 0.5, n * int(np.prod(shp))).reshape((n,) + shp)
        gen = self.F.Mt19937(19)
        self.m.train_stream(self._sv[:max(warmup, 1) * self.B], gen, self.B, self.lr)
        s = torch.cuda.ExternalStream(self.stream())
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record(s)
        self.m.train_stream(self._sv[:n], gen, self.B, self.lr)
        e1.record(s)
        torch.cuda.synchronize()
        return e0.elapsed_time(e1)

    def e2e_step(self):
        # crbm_cd_update(m, v0, lr, rng): the B*k*oh*ow draws generated on the device from the
        # caller's mt19937 (state up only when it changed, back every call)
        if getattr(self, "_gen", None) is None:
            self._gen = self.F.Mt19937(17)
        return self.F.crbm_cd_update(self.m, self.v0_h, self.lr, self._gen, self.Bg)

    def kernels_per_step(self):
        return _kernels(self.F._lib, "b2n_crbm_kernels_per_step", self.m.handle)

    @property
    def dtype(self):
        return "f32 (FFMA, one-launch step)" if self.kernels_per_step() == 1 else None

    def profile(self, steps):
        return _profile(self.F._lib, "b2n_crbm_profile", self.m.handle, steps, self.lr, self.Bg)

    def d2h_bytes(self):
        return 8


class NetWork:
    def __init__(self, name: str, dist: Dist, precision: int, nccl_id):
        from oracle import oracle as O
        from paper_1804_04512_b200 import configs as CF, fastnn as F
        from paper_1804_04512_b200.dp import shard_bounds
        self.name = name
        spec = CF.NET_CONFIGS[name]()
        self.Bg = spec["batch_size"]
        lo, hi = shard_bounds(self.Bg, dist.world, dist.rank)
        self.B = hi - lo
        per = int(np.prod(spec["input"]))
        classes = [d for d in spec["layers"] if d["kind"] == CF.DENSE][-1]["out"]
        rng = np.random.default_rng(1)
        if per * self.Bg <= 4_000_000:
            x = O.uniform_f32(1, self.Bg * per).reshape([self.Bg] + spec["input"])
        else:  # ImageNet-shape: numpy generator (the mt19937 stream is only needed for parity runs)
            x = rng.random((self.Bg, *spec["input"]), dtype=np.float32)
        lab = O.uniform_int(2, 0, classes - 1, self.Bg)
        x, lab = x[lo:hi], lab[lo:hi]
        self.net = F.build_network(spec, device=dist.local, precision=precision)
        if dist.world > 1:
            self.net.dp_init(nccl_id, dist.rank, dist.world)
        self.net.stage(x, lab)
        self.x_h = pinned((self.B, per), np.float32)
        self.x_h[:] = x.reshape(self.B, per)
        self.l_h = pinned((self.B,), np.int32)
        self.l_h[:] = lab
        self.F = F
        self.dist = dist
        desc = {"mlp": "MNIST-shape MLP 784-500-250-10 sigmoid, SGD+momentum",
                "mnist_cnn": "MNIST-shape CNN conv(8,5x5)+sigmoid+pool x2, dense 150, dense 10",
                "cifar_cnn": "CIFAR-shape CNN conv(12,5x5)+relu+pool x2, dense 64, dense 10",
                "imagenet_cnn": "ImageNet-shape CNN 5x conv(16,3x3,pad1)+relu+pool, dense 2048, dense 1000"}[name]
        self.config = {"workload": name, "model": desc, "global_batch": self.Bg, "local_batch": self.B,
                       "parallelism": f"dp{dist.world}", "lr": spec["lr"]}
        self.h2d = self.B * per * 4 + self.B * 4
        self.lr = spec["lr"]

    def stream(self):
        return self.net.stream_handle()

    def step(self, n=1):
        self.net.run_staged(n, self.Bg)

    def e2e_step(self):
        if self.dist.world > 1:
            self.net.forward_backward(self.x_h, self.l_h, self.Bg)
            self.net.apply_update()
            return None
        return self.F.train_minibatch_labels(self.net, self.x_h, self.l_h)

    def e2e_total(self, steps, warmup):
        """end to end through Network.train_stream (the loop of train_minibatch calls over host
        batches): every step's H2D (overlapped with the previous step) and loss read inside the
        timed region; distinct host batches (cycled when a step's input is large: ImageNet).
        Returns the device time of the whole run (ms) on the library stream."""
        if self.dist.world > 1:
            return None
        import torch
        per = self.x_h.shape[1]
        nb = max(2, min(steps, (256 << 20) // (per * self.B * 4)))
        if getattr(self, "_sx", None) is None or self._sx.shape[0] < nb * self.B:
            rng = np.random.default_rng(7)
            self._sx = pinned((nb * self.B, per), np.float32)
            self._sx[:] = rng.random((nb * self.B, per), dtype=np.float32)
            self._sl = pinned((nb * self.B,), np.int32)
            self._sl[:] = rng.integers(0, self.net.classes, nb * self.B, dtype=np.int32)

        def run(n):
            done = 0
            while done < n:
                k = min(nb, n - done)
                self.net.train_stream(self._sx[:k * self.B], self._sl[:k * self.B], self.B)
                done += k
        run(max(warmup, 2))
        s = torch.cuda.ExternalStream(self.stream())
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        self.dist.barrier()
        torch.cuda.synchronize()
        e0.record(s)
        run(steps)
        e1.record(s)
        torch.cuda.synchronize()
        self.dist.barrier()
        return self.dist.max(e0.elapsed_time(e1))

    def kernels_per_step(self):
        return self.net.kernels_per_step(self.B)

    def profile(self, steps):
        return _profile(self.F._lib, "b2n_net_profile", self.net.handle, self.B, steps)

    def d2h_bytes(self):
        return self.B * 8


def _kernels(lib, fn, h):
    import ctypes as C
    n = C.c_int()
    lib.call(fn, h, C.byref(n))
    return n.value


def _profile(lib, fn, h, *args):
    import ctypes as C
    max_ops = 256
    stats = (C.c_double * (4 * max_ops))()
    names = C.create_string_buffer(16384)
    n = C.c_int()
    lib.call(fn, h, *args, max_ops, stats, names, 16384, C.byref(n))
    nm = names.value.decode().split("\n")
    return [{"name": nm[i], "ms": stats[4 * i], "flops": stats[4 * i + 1], "bytes": stats[4 * i + 2],
             "kernels": int(stats[4 * i + 3])} for i in range(n.value)]


def make_work(name, dist, precision, nccl_id):
    if name == "crbm":
        return CrbmWork(dist, precision, nccl_id)
    return RbmWork(dist, precision, nccl_id) if name == "rbm" else NetWork(name, dist, precision, nccl_id)


# ----------------------------------------------------------------------------- timing
def time_steps(work, steps, warmup, dist, flush, e2e=False):
    """Per-step CUDA events on the library's stream, an L2 flush between steps (outside the
    events), max over ranks of the summed step time."""
    import torch
    s = torch.cuda.ExternalStream(work.stream())
    run = work.e2e_step if e2e else work.step
    for _ in range(warmup):
        run()
    torch.cuda.synchronize()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
    dist.barrier()
    torch.cuda.synchronize()
    for i in range(steps):
        with torch.cuda.stream(s):
            flush.zero_()
        ev[i][0].record(s)
        run()
        ev[i][1].record(s)
    torch.cuda.synchronize()
    dist.barrier()
    total_ms = sum(a.elapsed_time(b) for a, b in ev)
    return dist.max(total_ms)


def host_info() -> dict:
    """lscpu-style host description for the CPU baseline (model name, logical CPUs)."""
    model = None
    try:
        for ln in Path("/proc/cpuinfo").read_text().splitlines():
            if ln.startswith("model name"):
                model = ln.split(":", 1)[1].strip()
                break
    except Exception:
        pass
    import platform
    return {"cpu_model": model or platform.processor() or platform.machine(), "logical_cpus": os.cpu_count()}


_TF32 = {}


def measure_tf32_peak(dev: int) -> dict:
    """the TF32 tensor peak measured on this box (not assumed bf16/2): cuBLAS fp32 GEMM
    with TF32 math, 8192^3, best of 5 after warm-up (a measurement of the hardware, outside every
    timed region). 3xTF32 issues three TF32 products per fp32 product, so its peak is /3."""
    if dev in _TF32:
        return _TF32[dev]
    import torch
    n = 8192
    prev = torch.backends.cuda.matmul.allow_tf32
    try:
        torch.backends.cuda.matmul.allow_tf32 = True
        a = torch.randn(n, n, device=f"cuda:{dev}")
        b = torch.randn(n, n, device=f"cuda:{dev}")
        c = a @ b
        torch.cuda.synchronize()
        best = float("inf")
        for _ in range(5):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            torch.matmul(a, b, out=c)
            e1.record()
            torch.cuda.synchronize()
            best = min(best, e0.elapsed_time(e1))
        tf = 2.0 * n ** 3 / (best * 1e-3) / 1e12
        del a, b, c
        torch.cuda.empty_cache()
    finally:
        torch.backends.cuda.matmul.allow_tf32 = prev
    _TF32[dev] = {"tf32_tflops": round(tf, 1), "tf32x3_tflops": round(tf / 3.0, 1),
                  "how": "cuBLAS fp32 GEMM with TF32 math, 8192^3, best of 5 (CUDA events)"}
    return _TF32[dev]


def peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return d["hbm_gbs"], d["bf16_tflops"], "measured"
    return 6650.0, 1590.0, "fallback (B200_PROFILING.md)"


def roofline(prof, precision, tf32_meas=None, config=None):
    hbm, bf16, src = peaks()
    top = max(prof, key=lambda o: o["ms"])
    # tensor peak for the arithmetic in use: the measured TF32 rate (3xTF32 issues 3 products)
    if tf32_meas:
        tf32 = tf32_meas["tf32x3_tflops" if precision == "tf32x3" else "tf32_tflops"]
        tsrc = "measured " + tf32_meas["how"] + (" / 3 (3xTF32)" if precision == "tf32x3" else "")
    else:
        tf32 = bf16 / 2.0 / (3.0 if precision == "tf32x3" else 1.0)
        tsrc = src + f" (bf16 {bf16} TF/s -> tf32 /2" + (", 3xTF32 /3)" if precision == "tf32x3" else ")")
    ridge = tf32 * 1e12 / (hbm * 1e9)
    ai = top["flops"] / top["bytes"] if top["bytes"] else float("inf")
    sec = top["ms"] * 1e-3
    traffic = None
    tp = ROOT / "profiles" / "ncu_traffic.json"
    if tp.exists() and config:
        try:  # keyed "<config>/<op>" (profiles/summarize.py); null when that config's op was not captured
            traffic = json.loads(tp.read_text()).get(f"{config}/{top['name']}")
        except Exception:
            traffic = None
    if ai < ridge:
        ach = top["bytes"] / sec / 1e9
        return {"bound": "hbm", "kernel": top["name"], "achieved": round(ach, 2), "peak": hbm, "unit": "GB/s",
                "frac": round(ach / hbm, 5), "traffic": traffic, "algorithmic_bytes": top["bytes"],
                "flops": top["flops"], "avg_launch_us": round(top["ms"] * 1e3, 3), "peak_source": src,
                "tensor_peak_tflops": round(tf32, 1), "share_of_step": None}
    ach = top["flops"] / sec / 1e12
    return {"bound": "tensor", "kernel": top["name"], "achieved": round(ach, 3), "peak": round(tf32, 1),
            "unit": "TFLOP/s", "frac": round(ach / tf32, 5), "traffic": traffic, "algorithmic_bytes": top["bytes"],
            "flops": top["flops"], "avg_launch_us": round(top["ms"] * 1e3, 3),
            "peak_source": tsrc, "share_of_step": None}


def step_roofline(work, prof, precision, tf32, step_ms, config=None):
    """The dominant kernel's roofline (algorithmic bytes or FLOPs per launch / its event-timed launch
    duration) plus the whole step's: the planner's algorithmic bytes of every op / the step time,
    against the measured HBM peak, and the launch floor (dependent kernels x the measured 4.2 us
    single-kernel graph-launch latency, tools/launch_probe.cu)."""
    rl = roofline(prof, precision, tf32, config)
    prof_step = sum(o["ms"] for o in prof)
    rl["share_of_step"] = round(max(o["ms"] for o in prof) / prof_step, 4) if prof_step else None
    hbm = peaks()[0]
    step_bytes = sum(o["bytes"] for o in prof)
    rl["step_algorithmic_bytes"] = step_bytes
    rl["step_hbm_frac"] = round(step_bytes / (step_ms * 1e-3) / 1e9 / hbm, 5)
    rl["launch_floor_us"] = round(work.kernels_per_step() * 4.2, 2)
    rl["step_us"] = round(step_ms * 1e3, 2)
    return rl


# ----------------------------------------------------------------------------- CPU reference
def cpu_reference(name: str, budget_s: float, min_steps: int = 2, max_steps: int | None = None,
                  warmup_s: float = 0.0, warmup_min: int = 1, exact_steps: int | None = None):
    """Time the reference's own step on this host: oracle/_ref when built (kind 'reference'),
    else the oracle restatement (kind 'port'). Warm-up: at least `warmup_min` steps and `warmup_s`
    seconds (thread pool, page faults, caches at steady state). Then either exactly `exact_steps`
    timed steps, or steps until `budget_s` seconds (>= min_steps, <= max_steps).
    Returns (samples/s, info dict)."""
    import ctypes as C
    from oracle import oracle as O
    from paper_1804_04512_b200 import configs as CF
    threads = os.cpu_count() or 1
    if O.ref_available():
        lib, kind = O.load("ref"), "reference"
        lib.ref_set_threads(threads)
        cores = lib.ref_thread_count()
    else:
        lib, kind, cores = O.load("oracle"), "port", 1
    if name == "rbm":
        c = CF.RBM
        B, H, V = c["batch_size"], c["hidden"], c["visible"]
        v0 = O.bernoulli_f32(3, 0.5, B * V).reshape(B, V)
        if kind == "reference":
            h = lib.ref_rbm_create(H, V, c["seed"], O.fptr(v0), B, 5)
            step = lambda: lib.ref_rbm_step(h, c["lr"])  # noqa: E731
            done = lambda: lib.ref_rbm_destroy(h)  # noqa: E731
        else:
            W = O.rbm_init(H, V, c["seed"])
            bv, bh = np.zeros(V, np.float32), np.zeros(H, np.float32)
            u = O.canonical_f64(5, B * H)
            step = lambda: lib.orc_rbm_cd1(H, V, O.fptr(W), O.fptr(bv), O.fptr(bh), O.fptr(v0), B, B, c["lr"],  # noqa
                                           O.dptr(u), None, None, None, None, None, None, None)
            done = lambda: None  # noqa: E731
        what = "cd_k_update(k=1)"
    elif name == "crbm":
        c = CF.CRBM
        B = c["batch_size"]
        shp = (c["c_in"], c["h"], c["w"], c["k"], c["kh"], c["kw"])
        v0 = O.bernoulli_f32(3, 0.5, B * c["c_in"] * c["h"] * c["w"])
        if kind == "reference":
            h = lib.ref_crbm_create(*shp, c["seed"], O.fptr(v0), B, 5)
            step = lambda: lib.ref_crbm_step(h, c["lr"])  # noqa: E731
            done = lambda: lib.ref_crbm_destroy(h)  # noqa: E731
            what = "crbm_cd_update"
        else:
            ker = O.crbm_init(c["c_in"], c["h"], c["w"], c["k"], c["kh"], c["kw"], c["seed"])
            u = O.canonical_f64(5, B * c["k"] * (c["h"] - c["kh"] + 1) * (c["w"] - c["kw"] + 1))
            v4 = v0.reshape(B, c["c_in"], c["h"], c["w"])
            step = lambda: O.crbm_cd1(ker, np.zeros(c["c_in"], np.float32), np.zeros(c["k"], np.float32), v4,  # noqa
                                      c["lr"], u)
            done = lambda: None  # noqa: E731
            what = "oracle crbm_cd1"
    else:
        spec = CF.NET_CONFIGS[name]()
        B = spec["batch_size"]
        per = int(np.prod(spec["input"]))
        classes = [d for d in spec["layers"] if d["kind"] == CF.DENSE][-1]["out"]
        x = np.random.default_rng(1).random((B, per), dtype=np.float32)
        lab = O.uniform_int(2, 0, classes - 1, B)
        net = O.Net(spec, "ref" if kind == "reference" else "oracle")
        if kind == "reference":
            prepared = lib.ref_make_batch(net.h, O.fptr(x), O.iptr(lab), B)
            step = lambda: lib.ref_net_train_prepared(net.h, prepared)  # noqa: E731
            done = lambda: lib.ref_free_batch(prepared)  # noqa: E731
            what = "train_minibatch" + (" (pad=1 composite, SURVEY 8(c))" if name == "imagenet_cnn" else "")
        else:
            step = lambda: net.train_minibatch(x, lab)  # noqa: E731
            done = lambda: None  # noqa: E731
            what = "oracle train_minibatch"
    nw, t0 = 0, time.perf_counter()
    while nw < warmup_min or time.perf_counter() - t0 < warmup_s:
        step()
        nw += 1
    n, t0 = 0, time.perf_counter()
    while True:
        step()
        n += 1
        el = time.perf_counter() - t0
        if exact_steps is not None:
            if n >= exact_steps:
                break
        elif (el >= budget_s and n >= min_steps) or (max_steps and n >= max_steps):
            break
    done()
    return B * n / el, {"kind": kind, "cores": cores, "steps": n, "seconds": round(el, 3), "warmup_steps": nw,
                        "sample": f"{n} x {what}, global batch {B}, {cores} host threads, after {nw} warm-up steps"}


# ----------------------------------------------------------------------------- main
def fit_epochs(dev, precision):
    """one fastnn::fit epoch (network.hpp:488-511) over a synthetic dataset of the
    real dataset's size held in HBM (MNIST 60000, CIFAR-10 50000), through the public fit() API;
    samples/s from the epoch's batch-loop seconds as the reference reports them, plus the
    evaluate() pass fit runs afterwards."""
    from paper_1804_04512_b200 import configs as CF, fastnn as F
    out = {}
    for name, N in [("mlp", 60000), ("mnist_cnn", 60000), ("cifar_cnn", 50000)]:
        try:
            spec = CF.NET_CONFIGS[name]()
            rng = np.random.default_rng(3)
            x = rng.random((N, *spec["input"]), dtype=np.float32)
            lab = rng.integers(0, 10, N).astype(np.int32)
            net = F.build_network(spec, device=dev, precision=precision)
            F.fit(net, x[:spec["batch_size"] * 4], lab[:spec["batch_size"] * 4], 1)  # plans + graphs
            t0 = time.perf_counter()
            rep = F.fit(net, x, lab, 2)
            wall = time.perf_counter() - t0
            ep = rep.epochs[-1]
            out[name] = {"samples": N, "batch": spec["batch_size"], "epoch_s": round(ep.seconds, 5),
                         "samples_per_s": round(N / ep.seconds, 1), "loss": round(ep.loss, 5),
                         "train_accuracy": ep.accuracy, "fit_wall_s_2_epochs_incl_upload_and_eval": round(wall, 4)}
            del net
        except Exception as ex:
            out[name] = {"unavailable": f"{type(ex).__name__}: {ex}"[:200]}
    return out


def main():
    a = parse()
    dist = Dist()
    if a.impl == "reference":
        if dist.rank != 0:
            return
        name = a.config
        # steady state: >= max(W, 1) warm-up steps and >= 1.5 s of them, then exactly K timed steps
        v, info = cpu_reference(name, budget_s=0.0, warmup_s=1.5 if name != "imagenet_cnn" else 0.0,
                                warmup_min=max(a.warmup, 1) if name != "imagenet_cnn" else 1, exact_steps=a.steps)
        line = {"metric": "train samples/s", "value": round(v, 3), "unit": "samples/s", "n_gpus": a.gpus,
                "steps": info["steps"], "warmup": info["warmup_steps"],
                "ms_per_step": round(info["seconds"] * 1e3 / info["steps"], 3),
                "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f32",
                "data": "synthetic", "impl": "reference",
                "config": {"workload": {"rbm": "mnist_rbm_cd1", "crbm": "mnist_crbm_cd1"}.get(name, name),
                           "global_batch": 100 if name != "imagenet_cnn" else 128, "host": host_info()},
                "cpu_baseline": {"value": round(v, 3), "unit": "samples/s", "cores": info["cores"],
                                 "kind": info["kind"], "sample": info["sample"]},
                "e2e": {"value": round(v, 3), "unit": "samples/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
        print(json.dumps(line), flush=True)
        return

    import torch
    dist.init()
    dev = dist.local
    torch.cuda.set_device(dev)
    from paper_1804_04512_b200 import fastnn as F
    precision = F.TF32X3 if a.precision == "tf32x3" else F.TF32
    nccl_id = None
    if dist.world > 1:
        nccl_id = dist.bcast_bytes(F.nccl_unique_id() if dist.rank == 0 else None)
    flush = torch.empty(FLUSH_BYTES // 4, dtype=torch.float32, device=f"cuda:{dev}")
    work = make_work(a.config, dist, precision, nccl_id)
    if a.profile_only:
        work.step(a.warmup + a.steps)
        torch.cuda.synchronize()
        return
    # ramp clocks with a short untimed burst, then the timed regions under the clock sampler
    work.step(max(a.warmup, 3))
    torch.cuda.synchronize()
    t_end = time.perf_counter() + 0.3
    while time.perf_counter() < t_end:
        work.step(50)
        torch.cuda.synchronize()
    with ClockSampler(dev) as clk:
        flushed_ms = time_steps(work, a.steps, a.warmup, dist, flush)
        total_ms = work.value_total(a.steps, a.warmup, flush) if hasattr(work, "value_total") else None
        value_mode = "stream"
        if total_ms is None:
            total_ms, value_mode = flushed_ms, "flushed"
        e2e_ms = work.e2e_total(a.steps, max(a.warmup // 2, 3)) if hasattr(work, "e2e_total") else None
        e2e_mode = "stream"
        if e2e_ms is None:
            e2e_ms = time_steps(work, a.steps, max(a.warmup // 2, 3), dist, flush, e2e=True)
            e2e_mode = "per-call"
    prof = work.profile(max(min(a.steps, 50), 5))
    step_ms = total_ms / a.steps
    value = work.Bg * a.steps / (total_ms * 1e-3)
    e2e_val = work.Bg * a.steps / (e2e_ms * 1e-3)
    tf32 = measure_tf32_peak(dev)
    rl = step_roofline(work, prof, a.precision, tf32, step_ms, a.config)
    line = {"metric": "train samples/s", "value": round(value, 2), "unit": "samples/s", "n_gpus": dist.world,
            "steps": a.steps, "warmup": a.warmup, "ms_per_step": round(step_ms, 5), "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": getattr(work, "dtype", None) or (
                "f32 (3xTF32 tensor-core GEMMs)" if a.precision == "tf32x3" else "f32 (1xTF32 tensor-core GEMMs)"),
            "data": "synthetic",
            "config": dict(work.config, l2=(
                "flushed before the timed region (512 MiB write), then consecutive steps over %d distinct "
                "device-resident batches (%.0f MB), none read twice" % (a.steps, getattr(work, "value_bytes", 0) / 1e6)
                if value_mode == "stream" else
                "flushed between timed steps (512 MiB write)"), precision=a.precision),
            "value_flushed_per_step": {"value": round(work.Bg * a.steps / (flushed_ms * 1e-3), 2),
                                       "ms_per_step": round(flushed_ms / a.steps, 5),
                                       "how": "one step per timed region, 512 MiB L2 flush before each"},
            "e2e": {"value": round(e2e_val, 2), "unit": "samples/s", "h2d_bytes_per_step": work.h2d,
                    "d2h_bytes_per_step": work.d2h_bytes(), "ms_per_step": round(e2e_ms / a.steps, 5),
                    "api": ("Rbm.train_stream: one call over `steps` distinct pinned host batches (143 MB at 200 "
                            "steps, > L2) / Network.train_stream, each step's H2D overlapped with the previous "
                            "step, per-step result read back" if e2e_mode == "stream" else "one public-API step call per step (H2D, step, "
                            "result read), L2 flushed between steps")},
            # the `value` region's launches: the step kernels (+ the streamed loop's v0 staging kernel per step)
            "gpu_launches": (work.stream_launches_per_step() if value_mode == "stream" and
                             hasattr(work, "stream_launches_per_step") else work.kernels_per_step()) * a.steps,
            "kernels_per_step": work.kernels_per_step(),
            "roofline": rl,
            "tensor_peaks": tf32,
            "step_profile": [{k: (round(v, 5) if isinstance(v, float) else v) for k, v in o.items()} for o in prof],
            "clocks": clk.summary()}
    if not a.no_others:
        others = {}
        for name in ["rbm", "mlp", "mnist_cnn", "cifar_cnn", "imagenet_cnn", "crbm"]:
            if name == a.config:
                continue
            try:
                w = make_work(name, dist, precision, nccl_id)
                n = 20 if name == "imagenet_cnn" else 100
                ms = time_steps(w, n, 5, dist, flush)
                e2 = w.e2e_total(max(n // 2, 5), 2) if hasattr(w, "e2e_total") else None
                if e2 is None:
                    e2 = time_steps(w, max(n // 2, 5), 2, dist, flush, e2e=True)
                wprof = w.profile(10 if name == "imagenet_cnn" else 30)
                others[name] = {"value": round(w.Bg * n / (ms * 1e-3), 2), "unit": "samples/s",
                                "ms_per_step": round(ms / n, 5),
                                "e2e": round(w.Bg * max(n // 2, 5) / (e2 * 1e-3), 2),
                                "kernels_per_step": w.kernels_per_step(),
                                "roofline": step_roofline(w, wprof, a.precision, tf32, ms / n, name)}
                if dist.rank == 0 and dist.world == 1:  # the reference's own step beside every config
                    big = name == "imagenet_cnn"
                    cv, ci = cpu_reference(name, 0.0 if big else 3.0, min_steps=1 if big else 2,
                                           warmup_s=0.0 if big else 0.5)
                    others[name]["cpu_baseline"] = {"value": round(cv, 2), "unit": "samples/s",
                                                    "cores": ci["cores"], "kind": ci["kind"], "sample": ci["sample"]}
                del w
            except Exception as ex:  # a config the build does not cover yet is reported, not hidden
                others[name] = {"unavailable": f"{type(ex).__name__}: {ex}"[:200]}
        line["other_configs"] = others
    if dist.world == 1 and not a.no_others:
        line["fit_epoch"] = fit_epochs(dev, precision)
    if dist.rank == 0 and dist.world == 1:
        v, info = cpu_reference(a.config, a.cpu_budget, warmup_s=1.5)
        line["cpu_baseline"] = {"value": round(v, 2), "unit": "samples/s", "cores": info["cores"],
                                "kind": info["kind"], "sample": info["sample"], "host": host_info()}
    if dist.rank == 0:
        print(json.dumps(line), flush=True)
    if dist.pg:
        dist.pg.destroy_process_group()


if __name__ == "__main__":
    main()
