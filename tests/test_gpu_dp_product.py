"""Data-parallel execution of the PRODUCT library (libb200nn) beyond a 1-rank communicator
(the reference has none). Only one GPU exists here, so:
  * shard sums on one GPU: forward_backward / the RBM's gradient-only step over the shards of a global
    batch (batch_global = B) sum to the full-batch gradients -- for every BASELINE net config,
    including the ImageNet-shape 16-image shard the 8-GPU split runs;
  * world 2 through gloo: two processes on the same GPU each step their shard with the library, the
    library's packed gradients are allreduced by gloo between them (host round trip in place of
    NCCL), the library applies the update, and both replicas must equal the single-process
    full-batch step and stay bitwise in sync. This is the chain the NCCL step graph runs
    (forward_backward -> allreduce(G) -> packed SGD; RBM: fused CD-1 (raw sums) -> allreduce ->
    W += lr/B * G), with the collective swapped."""
import os
import socket

import numpy as np
import pytest

from conftest import norm_err
from oracle import oracle as O
from paper_1804_04512_b200 import configs as CF
from paper_1804_04512_b200.dp import shard_bounds

pytestmark = pytest.mark.gpu


def _net_inputs(name, B):
    spec = CF.NET_CONFIGS[name](B)
    classes = [d for d in spec["layers"] if d["kind"] == CF.DENSE][-1]["out"]
    x = O.uniform_f32(1, B * int(np.prod(spec["input"]))).reshape([B] + spec["input"])
    lab = O.uniform_int(2, 0, classes - 1, B)
    return spec, x, lab


@pytest.mark.parametrize("name,B,world", [("mlp", 100, 8), ("mnist_cnn", 100, 8), ("cifar_cnn", 100, 3),
                                          ("imagenet_cnn", 32, 2)])
def test_net_shard_sum_equals_full_batch(gpu, name, B, world):
    """sum over shards of forward_backward(shard, batch_global=B) == forward_backward(full batch)"""
    from paper_1804_04512_b200 import fastnn as F
    spec, x, lab = _net_inputs(name, B)
    full = F.build_network(spec)
    lf = full.forward_backward(x, lab)
    gfull = [full.get_param(i, F.GRAD).ravel() for i in range(full.num_params())]
    net = F.build_network(spec)
    gsum = [np.zeros_like(g, np.float64) for g in gfull]
    lsum = 0.0
    for r in range(world):
        lo, hi = shard_bounds(B, world, r)
        lsum += net.forward_backward(x[lo:hi], lab[lo:hi], B)
        for i in range(net.num_params()):
            gsum[i] += net.get_param(i, F.GRAD).ravel()
    assert abs(lsum - lf) <= 1e-6 * abs(lf)
    for i, (a, b) in enumerate(zip(gsum, gfull)):
        assert norm_err(a, b) < 1e-5, (name, i)


def test_rbm_grad_only_shards_sum_to_full_step(gpu):
    """the fused CD-1 kernel in gradient-only mode (what each rank runs before the allreduce):
    the shards' raw sums add up to the full batch's, and apply_update reproduces the fused
    single-GPU step"""
    from paper_1804_04512_b200 import fastnn as F
    B, H, V, lr = 100, 500, 784, 0.1
    v0 = O.bernoulli_f32(3, 0.5, B * V).reshape(B, V)
    u = O.canonical_f64(5, B * H).reshape(B, H)
    full = F.Rbm(H, V)
    full.init(42)
    rf = F.cd_k_update(full, v0, 1, lr, u)
    hs_full = full.last_states(B)[1]
    r = F.Rbm(H, V)
    r.init(42)
    r.set_grad_only(True)
    acc = [np.zeros((H, V)), np.zeros(V), np.zeros(H)]
    rsum, hs_sh = 0.0, []
    for k in range(4):
        lo, hi = shard_bounds(B, 4, k)
        rsum += F.cd_k_update(r, v0[lo:hi], 1, lr, u[lo:hi], batch_global=B)
        hs_sh.append(r.last_states(hi - lo)[1])
        assert r.kernels_per_step() == 1  # the fused kernel, not the split GEMMs
        for a, g in zip(acc, r.get_grad()):
            a += g
    w_before = r.get()[0]
    np.testing.assert_array_equal(w_before, O.rbm_init(H, V, 42))  # gradient-only: W untouched
    flips = int((np.concatenate(hs_sh) != hs_full).sum())
    assert flips <= 2, flips  # same probabilities up to the summation order of a smaller batch
    r.set_grad(*[a.astype(np.float32) for a in acc])
    r.apply_update(lr, B)
    wg, bvg, bhg = r.get()
    wf, bvf, bhf = full.get()
    W0 = O.rbm_init(H, V, 42)
    tol = 1e-5 if flips == 0 else 1e-3
    assert norm_err(wg - W0, wf - W0) < tol and norm_err(bvg, bvf) < tol and norm_err(bhg, bhf) < tol
    assert abs(rsum - rf) <= 1e-6 * rf


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, cfg, q):
    import sys
    from pathlib import Path
    root = Path(__file__).resolve().parents[1]
    sys.path.insert(0, str(root))
    sys.path.insert(0, str(root / "tests"))
    import torch
    import torch.distributed as dist
    from paper_1804_04512_b200 import fastnn as F
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        if cfg == "rbm":
            B, H, V, lr = 100, 500, 784, 0.1
            v0 = O.bernoulli_f32(3, 0.5, B * V).reshape(B, V)
            u = O.canonical_f64(5, B * H).reshape(B, H)
            lo, hi = shard_bounds(B, world, rank)
            rbm = F.Rbm(H, V)
            rbm.init(42)
            rbm.set_grad_only(True)
            out = []
            for _step in range(2):
                rec = torch.tensor([F.cd_k_update(rbm, v0[lo:hi], 1, lr, u[lo:hi], batch_global=B)],
                                   dtype=torch.float64)
                g = [torch.from_numpy(a.copy()) for a in rbm.get_grad()]
                flat = torch.cat([t.ravel() for t in g])
                dist.all_reduce(flat)  # the packed-gradient allreduce (NCCL in the product's step graph)
                dist.all_reduce(rec)
                n0, n1 = g[0].numel(), g[1].numel()
                rbm.set_grad(flat[:n0].numpy().reshape(H, V), flat[n0:n0 + n1].numpy(), flat[n0 + n1:].numpy())
                rbm.apply_update(lr, B)
                out.append(rec.item())
            params = torch.from_numpy(np.concatenate([a.ravel() for a in rbm.get()]))
        else:
            spec, x, lab = _net_inputs(cfg, 40)
            B = 40
            lo, hi = shard_bounds(B, world, rank)
            net = F.build_network(spec)
            out = []
            for _step in range(2):
                loss = torch.tensor([net.forward_backward(x[lo:hi], lab[lo:hi], B)], dtype=torch.float64)
                grads = [net.get_param(i, F.GRAD) for i in range(net.num_params())]
                flat = torch.from_numpy(np.concatenate([g.ravel() for g in grads]))
                dist.all_reduce(flat)
                dist.all_reduce(loss)
                off = 0
                for i, g in enumerate(grads):
                    net.set_param(i, flat[off:off + g.size].numpy().reshape(g.shape), F.GRAD)
                    off += g.size
                net.apply_update()  # the library's packed SGD kernel, identical on every replica
                out.append(loss.item())
            params = torch.from_numpy(np.concatenate([net.get_param(i).ravel() for i in range(net.num_params())]))
        gathered = [torch.zeros_like(params) for _ in range(world)]
        dist.all_gather(gathered, params)
        if rank == 0:
            q.put((out, gathered[0].numpy(), float((gathered[0] - gathered[1]).abs().max())))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("cfg", ["mlp", "mnist_cnn", "rbm"])
def test_world2_gloo_product_step(gpu, cfg):
    import torch.multiprocessing as mp
    from paper_1804_04512_b200 import fastnn as F
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, cfg, q)) for r in range(2)]
    for p in procs:
        p.start()
    losses, params, gap = q.get(timeout=300)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    assert gap == 0.0  # replicas bitwise in sync
    if cfg == "rbm":
        B, H, V = 100, 500, 784
        v0 = O.bernoulli_f32(3, 0.5, B * V).reshape(B, V)
        u = O.canonical_f64(5, B * H).reshape(B, H)
        ref = F.Rbm(H, V)
        ref.init(42)
        rec = [F.cd_k_update(ref, v0, 1, 0.1, u) for _ in range(2)]
        want = np.concatenate([a.ravel() for a in ref.get()])
        for a, b in zip(losses, rec):
            assert abs(a - b) <= 1e-5 * b
        assert norm_err(params, want) < 1e-4
    else:
        spec, x, lab = _net_inputs(cfg, 40)
        ref = F.build_network(spec)
        lf = [F.train_minibatch_labels(ref, x, lab) for _ in range(2)]
        want = np.concatenate([ref.get_param(i).ravel() for i in range(ref.num_params())])
        for a, b in zip(losses, lf):
            assert abs(a - b) <= 1e-5 * b
        assert norm_err(params, want) < 1e-5
