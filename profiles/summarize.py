"""Summarise the ncu captures of profiles/capture.sh into committed evidence.

    python profiles/summarize.py r1      # reads gpurun_out/r1_*, writes profiles/r1_*.md + ncu_traffic.json

Per kernel: duration, DRAM read+write bytes (-> `traffic` in bench.py's roofline), achieved DRAM
throughput, tensor-pipe activity, SM throughput, registers, and the SASS proof of tcgen05/TMA.
"""
from __future__ import annotations

import csv
import io
import json
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
OUT = ROOT / "gpurun_out"
PROF = ROOT / "profiles"

METRICS = {
    "dur_us": "gpu__time_duration.sum",
    "dram_read": "dram__bytes_read.sum",
    "dram_write": "dram__bytes_write.sum",
    "dram_pct": "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "tensor_pct": "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
    "sm_pct": "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "regs": "launch__registers_per_thread",
    "grid": "launch__grid_size",
}
UNIT_SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "usecond": 1, "nsecond": 1e-3, "msecond": 1e3}

CRBM_SPLIT = ["crbm.hidden+sample", "crbm.visible+stats", "crbm.neg_hidden", "crbm.stats", "crbm.update"]
RBM_STEP = ["rbm.hidden+sample", "rbm.visible+recon", "rbm.neg_hidden", "rbm.dW+update"]
# launch order of the halo-tile conv kernels in one ImageNet-shape step (capture.sh)
IMAGENET_CONV = [f"conv{i}.fwd" for i in range(5)] + [x for i in (4, 3, 2, 1) for x in (f"conv{i}.dgrad", f"conv{i}.wgrad")] + ["conv0.wgrad"]


def raw_rows(rep: Path):
    csvp = rep.with_suffix(".raw.csv")  # capture.sh exports the raw page on the box (reports are large)
    if csvp.exists():
        txt = csvp.read_text()
    else:
        txt = subprocess.run(["ncu", "-i", str(rep), "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    head, units = rows[0], rows[1]
    out = []
    for r in rows[2:]:
        d = {"kernel": r[head.index("Kernel Name")]}
        for k, m in METRICS.items():
            if m in head:
                i = head.index(m)
                try:
                    v = float(r[i].replace(",", ""))
                except ValueError:
                    v = None
                if v is not None:
                    v *= UNIT_SCALE.get(units[i], 1)
                d[k] = v
        out.append(d)
    return out


def launch_share(csv_path: Path):
    rows = [r for r in csv.reader(open(csv_path)) if r and not r[0].startswith("==")]
    head = rows[0]
    ki, vi, ui = head.index("Kernel Name"), head.index("Metric Value"), head.index("Metric Unit")
    mi = head.index("Metric Name") if "Metric Name" in head else None
    agg = {}
    for r in rows[1:]:
        if mi is not None and r[mi] != "gpu__time_duration.sum":
            continue
        v = float(r[vi].replace(",", ""))
        t = v * {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}.get(r[ui], 1.0)
        name = r[ki].split("(")[0]
        agg.setdefault(name, [0, 0.0])
        agg[name][0] += 1
        agg[name][1] += t
    return agg


def launch_bytes(csv_path: Path):
    """[(kernel name, DRAM read + write bytes)] per launch, in launch order"""
    rows = [r for r in csv.reader(open(csv_path)) if r and not r[0].startswith("==")]
    head = rows[0]
    ki, vi, mi, ii = head.index("Kernel Name"), head.index("Metric Value"), head.index("Metric Name"), head.index("ID")
    ui = head.index("Metric Unit")
    acc, order = {}, []
    for r in rows[1:]:
        if r[mi] not in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
            continue
        v = float(r[vi].replace(",", "")) * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(r[ui], 1)
        if r[ii] not in acc:
            acc[r[ii]] = [r[ki], 0.0]
            order.append(r[ii])
        acc[r[ii]][1] += v
    return [tuple(acc[i]) for i in order]


def main(tag: str):
    lines = [f"# ncu summary, round tag `{tag}` (B200, `--clock-control none`)", "",
             "Captured with `profiles/capture.sh` under gpurun; numbers from single-kernel replay",
             "(cold-cache, serialised): compare SHARES with bench.py's live CUDA-event timings, not absolutes.", ""]
    traffic = {}
    for rep, names, title, cfg in [(OUT / f"{tag}_rbm_full.ncu-rep", ["rbm.cd1_fused"],
                               "RBM CD-1 step (headline): the fused single-kernel step", "rbm"),
                              (OUT / f"{tag}_rbm_split_full.ncu-rep", RBM_STEP,
                               "RBM CD-1 step, split path (4 GEMM launches; data-parallel mode, B2N_RBM_FUSED=0)", None),
                              (OUT / f"{tag}_crbm_full.ncu-rep", ["crbm.cd1_fused"],
                               "Convolutional RBM CD-1 (SURVEY 8(f)4, MNIST shape): the one-launch step", "crbm"),
                              (OUT / f"{tag}_crbm_split_full.ncu-rep", CRBM_SPLIT,
                               "Convolutional RBM CD-1, split tensor-core path (B2N_CRBM_FUSED=0)", None),
                              (OUT / f"{tag}_imagenet_conv_full.ncu-rep", IMAGENET_CONV,
                               "ImageNet-shape CNN (batch 128): conv kernels of one step (convx forward, "
                               "tcgen05 dgrad, FFMA wgrad)", "imagenet_cnn"),
                              (OUT / f"{tag}_mt_full.ncu-rep", ["mt.words", "mt.canonical"],
                               "Device std::mt19937 stream: words (one-CTA wavefront) + canonical (grid)", "rng"),
                              (OUT / f"{tag}_bw_imagenet.ncu-rep", ["bw"] * 6,
                               "Bandwidth kernels of the ImageNet-shape step (softmax-xent rows, wgrad reduce + SGD, repack)", None),
                              (OUT / f"{tag}_bw_optim.ncu-rep", ["bw"] * 6,
                               "Packed optimizer passes (SGD in data-parallel mode, Adam/Adagrad/Adadelta)", None)]:
        if not rep.exists() and not rep.with_suffix(".raw.csv").exists():
            continue
        rows = raw_rows(rep)
        if names is IMAGENET_CONV:  # label by kernel kind, layers in launch order (fwd 0..4, bwd 4..0)
            names, fwd, bwd = [], 0, [4, 4, 4]
            for d in rows:
                k = d["kernel"]
                if k.startswith("void convx_fwd"):
                    names.append(f"conv{fwd}.fwd")
                    fwd += 1
                elif "convt_mma_kernel" in k:
                    names.append(f"conv{bwd[0]}.dgrad")
                    bwd[0] -= 1
                elif "convt_wgrad_kernel" in k:
                    names.append(f"conv{bwd[1]}.wgrad")
                    bwd[1] -= 1
                else:
                    names.append(f"conv{bwd[2]}.wgrad_reduce+sgd")
                    bwd[2] -= 1
        lines += [f"## {title}", "", "| op | kernel | us | DRAM rd+wr MB | DRAM GB/s | DRAM % | tensor-pipe % | SM % | regs | grid |",
                  "|---|---|---|---|---|---|---|---|---|---|"]
        for i, d in enumerate(rows):
            op = names[i] if i < len(names) else "?"
            tb = (d.get("dram_read") or 0) + (d.get("dram_write") or 0)
            # per launch, keyed "<config>/<op>" as bench.py's roofline `traffic` looks it up (the same op
            # name, e.g. conv1.dgrad, names different kernels in different configs)
            if cfg and op not in ("bw", "?"):
                traffic.setdefault(f"{cfg}/{op}", tb)
            gbs = tb / (d.get('dur_us') or 1e9) / 1e3
            lines.append(f"| {op} | `{d['kernel'][:60]}` | {d.get('dur_us', 0):.2f} | {tb / 1e6:.3f} | {gbs:.0f} | "
                         f"{d.get('dram_pct', 0):.1f} | {d.get('tensor_pct', 0):.1f} | {d.get('sm_pct', 0):.1f} | "
                         f"{d.get('regs', 0):.0f} | {d.get('grid', 0):.0f} |")
        lines.append("")
    for c in ["rbm", "mlp", "mnist_cnn", "cifar_cnn", "imagenet_cnn", "crbm"]:
        p = OUT / f"{tag}_launches_{c}.csv"
        if not p.exists():
            continue
        agg = launch_share(p)
        tot = sum(v[1] for v in agg.values())
        lines += [f"## launch list: `bench.py --profile-only --config {c}` (warm-up + 1 step)", "",
                  "| kernel | launches | total us | share |",
                  "|---|---|---|---|"]
        for k, (n, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
            lines.append(f"| `{k[:70]}` | {n} | {t:.1f} | {t / tot:.1%} |")
        lines.append("")
    lib = ROOT / "paper_1804_04512_b200" / "_build" / "libb200nn.so"
    if lib.exists():
        sass = subprocess.run(["cuobjdump", "-sass", str(lib)], capture_output=True, text=True).stdout
        import re
        counts = {m: len(re.findall(r"\b" + m + r"\b", sass))
                  for m in ["UTCHMMA", "UTMALDG", "UBLKCP", "LDTM", "STTM", "UTCBAR", "HMMA"]}
        lines += ["## SASS evidence (cuobjdump -sass libb200nn.so)", "",
                  "| mnemonic | count | meaning |", "|---|---|---|",
                  f"| UTCHMMA | {counts['UTCHMMA']} | tcgen05.mma (kind::tf32) |",
                  f"| UTMALDG | {counts['UTMALDG']} | TMA tensor loads |",
                  f"| UBLKCP | {counts['UBLKCP']} | cp.async.bulk (conv halo rows) |",
                  f"| STTM | {counts['STTM']} | tcgen05.st (conv accumulator re-zeroing) |",
                  f"| LDTM | {counts['LDTM']} | tcgen05.ld (TMEM -> registers) |",
                  f"| UTCBAR | {counts['UTCBAR']} | tcgen05.commit -> mbarrier |",
                  f"| HMMA | {counts['HMMA']} | legacy mma.sync (none expected) |", ""]
    (PROF / f"{tag}_ncu_summary.md").write_text("\n".join(lines) + "\n")
    # the dominant op of the small configs from their launch lists (DRAM bytes per launch, last step):
    # the one tcgen05 dgrad of the MNIST / CIFAR step (conv1.dgrad) and the MLP's first GEMM (dense0)
    for cfg, pick in [("mnist_cnn", ("conv1.dgrad", "convt_mma_kernel", -1)),
                      ("cifar_cnn", ("conv1.dgrad", "convt_mma_kernel", -1)),
                      ("mlp", ("dense0.fwd+act", "gemm_tc_kernel", -8))]:
        p = OUT / f"{tag}_launches_{cfg}.csv"
        if not p.exists():
            continue
        launches = launch_bytes(p)
        sel = [b for k, b in launches if pick[1] in k]
        if len(sel) >= -pick[2]:
            traffic[f"{cfg}/{pick[0]}"] = sel[pick[2]]
        if cfg != "mlp":  # the two conv weight gradients (+ reduce / SGD), conv1 then conv0 in the backward
            wg = [b for k, b in launches if "convt_wgrad_kernel" in k]
            rd = [b for k, b in launches if "convt_wgrad_reduce_kernel" in k]
            if len(wg) >= 2 and len(rd) >= 2:
                traffic[f"{cfg}/conv1.wgrad+sgd"] = wg[-2] + rd[-2]
                traffic[f"{cfg}/conv0.wgrad+sgd"] = wg[-1] + rd[-1]
    # bench.py's ops that are two launches: the FFMA weight gradient + its reduce/SGD pass
    for k in list(traffic):
        if k.endswith(".wgrad") and k + "_reduce+sgd" in traffic:
            traffic[k + "+sgd"] = traffic[k] + traffic[k + "_reduce+sgd"]
    (PROF / "ncu_traffic.json").write_text(json.dumps(traffic, indent=1) + "\n")
    print("\n".join(lines))


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "r1")
