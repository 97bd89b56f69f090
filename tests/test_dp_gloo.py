"""Data-parallel step logic at world_size 2 over gloo on CPU: contiguous shards,
dlogits scaled by the GLOBAL batch (network.hpp:430 would use the local one), one allreduce of the
packed gradients, an identical update on every replica -- checked against the full-batch step of
the oracle. The GPU path runs the same algebra with NCCL inside its step graph."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1804_04512_b200.dp import shard_bounds, shard_sizes


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, cfg, q):
    import sys
    from pathlib import Path
    sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
    from oracle import oracle as O
    from paper_1804_04512_b200 import configs as CF
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        if cfg == "rbm":
            H, V, B = 30, 50, 11
            W = O.rbm_init(H, V, 42)
            v0 = O.bernoulli_f32(3, 0.5, B * V).reshape(B, V)
            u = O.canonical_f64(5, B * H).reshape(B, H)
            lo, hi = shard_bounds(B, world, rank)
            _, _, _, _, ex = O.rbm_cd1(W, np.zeros(V, np.float32), np.zeros(H, np.float32), v0[lo:hi], 0.1, u[lo:hi],
                                       b_global=B, deltas=True)
            parts = [torch.from_numpy(ex[k].copy()) for k in ("dW", "dbv", "dbh")]
            for t in parts:
                dist.all_reduce(t)
            W1 = W + parts[0].numpy()
            if rank == 0:
                _, Wf, bvf, bhf, _ = O.rbm_cd1(W, np.zeros(V, np.float32), np.zeros(H, np.float32), v0, 0.1, u)
                q.put(("rbm", float(np.abs(W1 - Wf).max()), float(np.abs(parts[1].numpy() - bvf).max()),
                       float(np.abs(parts[2].numpy() - bhf).max())))
        else:
            spec = CF.NET_CONFIGS[cfg](20)
            B = 20
            per = int(np.prod(spec["input"]))
            x = O.uniform_f32(1, B * per).reshape([B] + spec["input"])
            lab = O.uniform_int(2, 0, 9, B)
            lo, hi = shard_bounds(B, world, rank)
            net = O.Net(spec)
            loss = torch.tensor([net.forward_backward(x[lo:hi], lab[lo:hi], b_global=B)], dtype=torch.float64)
            grads = [torch.from_numpy(net.get(i, 1)) for i in range(net.num_params())]
            flat = torch.cat(grads)
            dist.all_reduce(flat)  # the packed-buffer allreduce
            dist.all_reduce(loss)
            off = 0
            for i, gr in enumerate(grads):
                net.set(i, flat[off:off + gr.numel()].numpy(), which=1)
                off += gr.numel()
            net.apply()  # identical SGD on every replica
            params = torch.cat([torch.from_numpy(net.get(i)) for i in range(net.num_params())])
            gathered = [torch.zeros_like(params) for _ in range(world)]
            dist.all_gather(gathered, params)
            if rank == 0:
                full = O.Net(spec)
                lf = full.train_minibatch(x, lab)
                ref = torch.cat([torch.from_numpy(full.get(i)) for i in range(full.num_params())])
                den = float(ref.abs().max())
                q.put((cfg, float(abs(loss.item() - lf) / lf), float((gathered[0] - ref).abs().max()) / den,
                       float((gathered[0] - gathered[1]).abs().max())))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("cfg", ["mlp", "mnist_cnn", "rbm"])
def test_two_rank_step_equals_full_batch(cfg):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, cfg, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = q.get(timeout=240)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    if cfg == "rbm":
        _, dw, dbv, dbh = res
        assert dw < 1e-6 and dbv < 1e-6 and dbh < 1e-6
    else:
        _, dloss, dparam, replica_gap = res
        assert dloss < 1e-12 and dparam < 1e-6
        assert replica_gap == 0.0  # replicas stay bitwise in sync


def test_shard_bounds():
    assert shard_sizes(100, 8) == [13, 13, 13, 13, 12, 12, 12, 12]
    assert shard_sizes(128, 8) == [16] * 8
    assert shard_sizes(100, 1) == [100]
    for B in (1, 7, 100, 128):
        for w in (1, 2, 3, 4, 8):
            b = [shard_bounds(B, w, r) for r in range(w)]
            assert b[0][0] == 0 and b[-1][1] == B
            assert all(b[i][1] == b[i + 1][0] for i in range(w - 1))
