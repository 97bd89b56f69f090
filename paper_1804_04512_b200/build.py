"""Build libb200nn.so (the CUDA kernels + C ABI) in-tree for sm_100a with nvcc.

    python -m paper_1804_04512_b200.build [--verbose]

Each csrc/*.cu translation unit (C ABI + runtime, one per GEMM epilogue, one per conv mode) is
compiled in parallel to an object, then linked into paper_1804_04512_b200/_build/libb200nn.so
(git-ignored; travels to the GPU box with the snapshot). The CUDA runtime is linked statically so
the library does not depend on which libcudart a host process (e.g. torch) already loaded; NCCL is
dlopen'ed on first use.
"""
from __future__ import annotations

import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path

PKG = Path(__file__).resolve().parent
CSRC = PKG / "csrc"
OUT_DIR = PKG / "_build"
LIB = OUT_DIR / "libb200nn.so"
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "--expt-relaxed-constexpr", "-Xcompiler", "-fPIC"]


def sources() -> list[Path]:
    return sorted(CSRC.glob("*.cu")) + sorted(CSRC.glob("*.cuh")) + [PKG.parent / "include" / "b200nn.h"]


def up_to_date() -> bool:
    if not LIB.exists():
        return False
    t = LIB.stat().st_mtime
    return all(s.stat().st_mtime <= t for s in sources())


def _compile(src: Path, verbose: bool) -> tuple[Path, str]:
    obj = OUT_DIR / (src.stem + ".o")
    cmd = [NVCC, *ARCH, *FLAGS, "-c", str(src), "-o", str(obj)]
    if verbose:
        cmd.insert(1, "-Xptxas=-v")
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed on {src.name}:\n{r.stdout}{r.stderr}")
    return obj, r.stderr


def build(verbose: bool = False, force: bool = False) -> Path:
    if up_to_date() and not force:
        return LIB
    OUT_DIR.mkdir(exist_ok=True)
    units = sorted(CSRC.glob("*.cu"))
    with ThreadPoolExecutor(max_workers=min(len(units), os.cpu_count() or 4)) as ex:
        results = list(ex.map(lambda s: _compile(s, verbose), units))
    if verbose:
        for _, err in results:
            sys.stderr.write(err)
    cmd = [NVCC, *ARCH, "-shared", "-o", str(LIB) + ".tmp", *[str(o) for o, _ in results], "-ldl", "-lcuda"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError("nvcc link of libb200nn.so failed")
    os.replace(str(LIB) + ".tmp", LIB)
    return LIB


if __name__ == "__main__":
    build(verbose="--verbose" in sys.argv, force=True)
    print(LIB)
