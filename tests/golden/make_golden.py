"""Generate the golden fixtures that pin the oracle to the reference (run in the build container,
where /root/reference exists and oracle/_ref/libfastnn_ref.so is built by `make -C oracle`).

Every array here comes from the UNMODIFIED reference (fastnn headers compiled behind
oracle/ref_shim.cpp): build_network / train_minibatch (network.hpp:284, :463), gemm
(gemm.hpp:225), cd_k_update (energy.hpp:131), sgd_momentum_step (optim.hpp:69) and, for the
padded ImageNet-shaped net, the SURVEY 8(c) composite of reference primitives.

    python tests/golden/make_golden.py        # writes tests/golden/*.npz and full_size.json
    python tests/golden/make_golden.py fit    # only fit.npz (fit / evaluate / batch order)
    python tests/golden/make_golden.py checkpoint  # only *.fnn1 + checkpoint_errors.json
    python tests/golden/make_golden.py optim  # only optim.npz (Adagrad / Adadelta / Adam)
    python tests/golden/make_golden.py dbn    # only dbn.npz (dbn_pretrain)
    python tests/golden/make_golden.py crbm   # only crbm.npz (crbm_cd_update)
    python tests/golden/make_golden.py cdk    # only rbm_cdk.npz (cd_k_update, k = 2 and 3)
"""
from __future__ import annotations

import json
import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
ROOT = HERE.parents[1]
sys.path.insert(0, str(ROOT))

from oracle import oracle as O  # noqa: E402
from paper_1804_04512_b200 import configs as CF  # noqa: E402


def small_specs():
    mlp = {"input": [64], "layers": [CF.dense(64, 48), CF.sigmoid(), CF.dense(48, 24), CF.sigmoid(),
                                     CF.dense(24, 10), CF.softmax()], "lr": 0.1, "momentum": 0.9, "seed": 42}
    mnist = {"input": [1, 12, 12], "layers": [CF.conv(4, 3, 3), CF.sigmoid(), CF.maxpool(), CF.conv(4, 2, 2),
                                              CF.sigmoid(), CF.maxpool(), CF.dense(16, 12), CF.sigmoid(),
                                              CF.dense(12, 10), CF.softmax()], "lr": 0.1, "momentum": 0.9, "seed": 7}
    cifar = {"input": [3, 16, 16], "layers": [CF.conv(5, 5, 5), CF.relu(), CF.maxpool(), CF.conv(5, 3, 3),
                                              CF.relu(), CF.maxpool(), CF.dense(20, 8), CF.relu(),
                                              CF.dense(8, 10), CF.softmax()], "lr": 0.01, "momentum": 0.9,
             "seed": 11}
    imnet = {"input": [3, 16, 16], "layers": [CF.conv(4, 3, 3, 1), CF.relu(), CF.maxpool(), CF.conv(4, 3, 3, 1),
                                              CF.relu(), CF.maxpool(), CF.dense(64, 16), CF.relu(),
                                              CF.dense(16, 10), CF.softmax()], "lr": 0.05, "momentum": 0.9,
             "seed": 13}
    return {"mlp_small": (mlp, 12), "mnist_cnn_small": (mnist, 6), "cifar_cnn_small": (cifar, 5),
            "imagenet_cnn_small": (imnet, 3)}


def net_case(spec, B, steps=2):
    per = int(np.prod(spec["input"]))
    x = O.uniform_f32(101, B * per).reshape([B] + spec["input"])
    lab = O.uniform_int(102, 0, 9, B)
    ref = O.Net(spec, "ref")
    out = {"x": x, "labels": lab}
    for i in range(ref.num_params()):
        out[f"init{i}"] = ref.get(i)
    losses = []
    probs = np.zeros((B, 10), np.float32)
    losses.append(ref.forward_backward(x, lab, probs=probs))
    out["probs0"] = probs
    for i in range(ref.num_params()):
        out[f"grad{i}"] = ref.get(i, 1)
    ref.apply()
    for _ in range(steps - 1):
        losses.append(ref.train_minibatch(x, lab))
    for i in range(ref.num_params()):
        out[f"final{i}"] = ref.get(i)
        out[f"vel{i}"] = ref.get(i, 2)
    p, am = ref.forward(x)
    out["probs_final"], out["argmax_final"] = p, am
    out["losses"] = np.array(losses)
    return out


FIT_CASES = {  # name -> (small spec, dataset size, batch size, epochs); N % batch != 0 on purpose
    "mlp_small": (250, 32, 3),
    "mnist_cnn_small": (90, 20, 2),
}


def fit_cases():
    """fit / evaluate / BatchIterator order (network.hpp:474-511, data.hpp:224-266) from the reference."""
    out = {}
    for N, seed in [(250, 42), (90, 7), (1000, 3)]:
        for e in range(3):
            out[f"order_{N}_{seed}_{e}"] = O.batch_order(N, seed, e, "ref")
    specs = small_specs()
    for name, (N, B, epochs) in FIT_CASES.items():
        spec = specs[name][0]
        per = int(np.prod(spec["input"]))
        x = O.uniform_f32(201, N * per).reshape([N] + spec["input"])
        lab = O.uniform_int(202, 0, 9, N)
        ref = O.Net(spec, "ref")
        out[f"{name}_x"], out[f"{name}_labels"] = x, lab
        out[f"{name}_acc0"] = np.array([ref.evaluate(x, lab, B)])
        loss, acc = ref.fit(x, lab, B, spec["seed"], epochs)
        out[f"{name}_loss"], out[f"{name}_acc"] = loss, acc
        for i in range(ref.num_params()):
            out[f"{name}_final{i}"] = ref.get(i)
    np.savez_compressed(HERE / "fit.npz", **out)


def checkpoint_cases():
    """save_network bytes (network.hpp:552-573) of each small net after its two golden steps, plus
    the reference's error texts for malformed files (network.hpp:575-607)."""
    errs = {}
    for name in ["mlp_small", "mnist_cnn_small", "cifar_cnn_small"]:
        spec, _ = small_specs()[name]
        g = np.load(HERE / f"{name}.npz")
        ref = O.Net(spec, "ref")
        for _ in range(2):
            ref.train_minibatch(g["x"], g["labels"])
        path = HERE / f"{name}.fnn1"
        assert O.ref_checkpoint(ref, path) == ""
        data = path.read_bytes()
        cases = {"bad_magic": b"FNN2" + data[4:], "truncated": data[:-3], "empty": b"",
                 "layer_count": data[:4] + (99).to_bytes(4, "little") + data[8:],
                 "tag": data[:12] + b"x" + data[13:]}
        for case, blob in cases.items():
            tmp = HERE / "_tmp.fnn1"
            tmp.write_bytes(blob)
            errs[f"{name}:{case}"] = O.ref_checkpoint(ref, tmp, load=True)
            tmp.unlink()
        errs[f"{name}:missing"] = O.ref_checkpoint(ref, HERE / "_does_not_exist.fnn1", load=True)
    (HERE / "checkpoint_errors.json").write_text(json.dumps(errs, indent=1))


def optim_cases():
    """Adagrad / Adadelta / Adam (optim.hpp:83-137): 4 reference steps of two small nets, lr 0.01"""
    out = {}
    for name in ["mlp_small", "mnist_cnn_small"]:
        spec, _ = small_specs()[name]
        g = np.load(HERE / f"{name}.npz")
        for kind in (1, 2, 3):
            ref = O.Net(dict(spec, optimizer=kind, lr=0.01), "ref")
            out[f"{name}_{kind}_losses"] = np.array([ref.train_minibatch(g["x"], g["labels"]) for _ in range(4)])
            for i in range(ref.num_params()):
                for w in (0, 3, 4):
                    out[f"{name}_{kind}_{w}_{i}"] = ref.get(i, w)
    np.savez_compressed(HERE / "optim.npz", **out)


DBN_CASE = {"dims": [40, 24, 16], "n": 50, "epochs": 2, "lr": 0.1, "batch": 16, "seed": 5}


def dbn_case_inputs():
    c = DBN_CASE
    dims = c["dims"]
    stack = [(O.rbm_init(dims[l + 1], dims[l], 42 + l), O.uniform_f32(9 + l, dims[l], -0.1, 0.1),
              O.uniform_f32(19 + l, dims[l + 1], -0.1, 0.1)) for l in range(len(dims) - 1)]
    data = O.bernoulli_f32(3, 0.5, c["n"] * dims[0]).reshape(c["n"], dims[0])
    return stack, data


def dbn_cases():
    """the reference's dbn_pretrain (energy.hpp:208-240) on a 40-24-16 stack, 50 rows, batch 16
    (a partial last batch), 2 epochs, one mt19937(5) stream"""
    c = DBN_CASE
    stack, data = dbn_case_inputs()
    out, recon = O.ref_dbn_pretrain(stack, data, c["epochs"], c["lr"], c["batch"], c["seed"])
    g = {"recon": np.array(recon)}
    for l, (W, bv, bh) in enumerate(out):
        g[f"W{l}"], g[f"bv{l}"], g[f"bh{l}"] = W, bv, bh
    np.savez_compressed(HERE / "dbn.npz", **g)


# CRBM shapes (c, h, w, k, kh, kw, batch): the reference test's 1x4x4 / 3x3 single-kernel case
# (test_energy.cpp:374-435), the toy-image case (:437-464), the 1x1 dense-degenerate case
# (:466-503), a multi-channel rectangular case and an MNIST-shaped one
CRBM_CASES = [(1, 4, 4, 1, 3, 3, 1), (1, 6, 6, 4, 3, 3, 8), (3, 1, 1, 2, 1, 1, 4), (2, 10, 9, 5, 3, 2, 3),
              (1, 28, 28, 12, 5, 5, 4)]


def crbm_case_inputs(i):
    c, h, w, k, kh, kw, B = CRBM_CASES[i]
    ker = O.crbm_init(c, h, w, k, kh, kw, 42 + i, "ref")
    bv = O.uniform_f32(7 + i, c, -0.1, 0.1)
    bh = O.uniform_f32(8 + i, k, -0.1, 0.1)
    v0 = O.bernoulli_f32(3 + i, 0.5, B * c * h * w).reshape(B, c, h, w)
    return ker, bv, bh, v0


def crbm_cases():
    """the reference's crbm_cd_update (energy.hpp:333-376) on CRBM_CASES, std::mt19937(5 + i)"""
    g = {}
    for i in range(len(CRBM_CASES)):
        ker, bv, bh, v0 = crbm_case_inputs(i)
        recon, k1, bv1, bh1 = O.ref_crbm_cd(ker, bv, bh, v0, 0.1, 5 + i)
        g.update({f"ker{i}": ker, f"bv{i}": bv, f"bh{i}": bh, f"v0_{i}": v0, f"ker1_{i}": k1, f"bv1_{i}": bv1,
                  f"bh1_{i}": bh1, f"recon{i}": np.array([recon])})
    np.savez_compressed(HERE / "crbm.npz", **g)


CDK_CASES = [(2, 12, 40, 30), (3, 9, 24, 17)]  # (k, batch, hidden, visible)


def cdk_cases():
    """the reference's cd_k_update (energy.hpp:131-171) for k > 1 with std::mt19937(11 + i): the Gibbs
    chain resamples hs from each intermediate visible mean (k * B * H draws per step)"""
    g = {}
    for i, (k, B, H, V) in enumerate(CDK_CASES):
        W = O.rbm_init(H, V, 42 + i, "ref")
        bv = O.uniform_f32(7 + i, V, -0.1, 0.1)
        bh = O.uniform_f32(8 + i, H, -0.1, 0.1)
        v0 = O.bernoulli_f32(3 + i, 0.5, B * V).reshape(B, V)
        recon, W1, bv1, bh1 = O.ref_cd_k(W, bv, bh, v0, k, 0.1, 11 + i)
        g.update({f"W{i}": W, f"bv{i}": bv, f"bh{i}": bh, f"v0_{i}": v0, f"W1_{i}": W1, f"bv1_{i}": bv1,
                  f"bh1_{i}": bh1, f"recon{i}": np.array([recon]), f"k{i}": np.array([k])})
    np.savez_compressed(HERE / "rbm_cdk.npz", **g)


def main():
    if sys.argv[1:] == ["cdk"]:
        cdk_cases()
        print("cd-k fixtures written to", HERE)
        return
    if sys.argv[1:] == ["crbm"]:
        crbm_cases()
        print("crbm fixtures written to", HERE)
        return
    if sys.argv[1:] == ["dbn"]:
        dbn_cases()
        print("dbn fixtures written to", HERE)
        return
    if sys.argv[1:] == ["optim"]:
        optim_cases()
        print("optimizer fixtures written to", HERE)
        return
    if sys.argv[1:] == ["fit"]:
        fit_cases()
        print("fit fixtures written to", HERE)
        return
    if sys.argv[1:] == ["checkpoint"]:
        checkpoint_cases()
        print("checkpoint fixtures written to", HERE)
        return
    assert O.ref_available(), "build oracle/_ref first (make -C oracle) -- needs /root/reference"
    meta = {}
    rng = np.random.default_rng(2024)
    g = {}
    for ta in (0, 1):
        for tb in (0, 1):
            M, N, K = 13, 11, 17
            a = rng.standard_normal((K, M) if ta else (M, K)).astype(np.float32)
            b = rng.standard_normal((N, K) if tb else (K, N)).astype(np.float32)
            g[f"a_{ta}{tb}"], g[f"b_{ta}{tb}"] = a, b
            g[f"c_{ta}{tb}"] = O.gemm(ta, tb, a, b, "ref")
    np.savez_compressed(HERE / "gemm.npz", **g)
    for name, (spec, B) in small_specs().items():
        np.savez_compressed(HERE / f"{name}.npz", **net_case(spec, B))
        meta[name] = {"spec": spec, "batch": B}
    # RBM CD-1 (the reference consumes its own std::mt19937(seed); the oracle takes the same stream
    # as supplied uniforms)
    H, V, B = 24, 40, 8
    W = O.rbm_init(H, V, 42, "ref")
    v0 = O.bernoulli_f32(3, 0.5, B * V).reshape(B, V)
    bv = O.uniform_f32(9, V, -0.1, 0.1)
    bh = O.uniform_f32(10, H, -0.1, 0.1)
    recon, W1, bv1, bh1 = O.ref_cd_k(W, bv, bh, v0, 1, 0.1, 5)
    np.savez_compressed(HERE / "rbm.npz", W=W, bv=bv, bh=bh, v0=v0, W1=W1, bv1=bv1, bh1=bh1,
                        recon=np.array([recon]), rng_seed=np.array([5]))
    # SGD trace (acceptance.cpp:483-555 grads {0.3, -0.2, 0.05})
    p = np.array([1.0, 0, 0, 0], np.float32)
    v = np.zeros(4, np.float32)
    trace = []
    lib = O.load("ref")
    for gv in (0.3, -0.2, 0.05):
        gg = np.array([gv, 0, 0, 0], np.float32)
        lib.ref_sgd_momentum_step(O.fptr(p), O.fptr(v), O.fptr(gg), 4, 0.1, 0.9, 0.0)
        trace.append(p[0])
    np.savez_compressed(HERE / "sgd.npz", trace=np.array(trace, np.float32))
    # full-size checksums: one reference step of every config at its full batch (B=100; the
    # ImageNet-shaped composite at batch 2 to stay within seconds)
    full = {}
    for name in ["mlp", "mnist_cnn", "cifar_cnn", "imagenet_cnn"]:
        spec = CF.NET_CONFIGS[name](2 if name == "imagenet_cnn" else 100)
        B = spec["batch_size"]
        per = int(np.prod(spec["input"]))
        classes = [d for d in spec["layers"] if d["kind"] == CF.DENSE][-1]["out"]
        x = O.uniform_f32(1, B * per).reshape([B] + spec["input"])
        lab = O.uniform_int(2, 0, classes - 1, B)
        ref = O.Net(spec, "ref")
        loss = ref.train_minibatch(x, lab)
        full[name] = {"batch": B, "loss": loss,
                      "param_sums": [float(np.sum(ref.get(i).astype(np.float64))) for i in range(ref.num_params())],
                      "param_abs_sums": [float(np.sum(np.abs(ref.get(i).astype(np.float64))))
                                         for i in range(ref.num_params())]}
    c = CF.RBM
    W = O.rbm_init(c["hidden"], c["visible"], c["seed"], "ref")
    v0 = O.bernoulli_f32(3, 0.5, c["batch_size"] * c["visible"]).reshape(c["batch_size"], c["visible"])
    recon, W1, bv1, bh1 = O.ref_cd_k(W, np.zeros(c["visible"], np.float32), np.zeros(c["hidden"], np.float32), v0,
                                     1, c["lr"], 5)
    full["rbm"] = {"recon": recon, "w_sum": float(np.sum(W1.astype(np.float64))),
                   "bv_sum": float(np.sum(bv1.astype(np.float64))), "bh_sum": float(np.sum(bh1.astype(np.float64)))}
    (HERE / "full_size.json").write_text(json.dumps(full, indent=1))
    (HERE / "meta.json").write_text(json.dumps(meta, indent=1))
    fit_cases()
    checkpoint_cases()
    optim_cases()
    dbn_cases()
    crbm_cases()
    print("golden fixtures written to", HERE)


if __name__ == "__main__":
    main()
