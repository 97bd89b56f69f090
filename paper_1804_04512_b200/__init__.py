"""B200-native data-parallel training step of DLL (arXiv 1804.04512).

The product is libb200nn.so (paper_1804_04512_b200/csrc -> _build/, C ABI in include/b200nn.h):
tcgen05 tensor-core GEMM / implicit-GEMM conv kernels with fused epilogues, bandwidth kernels and
NCCL data parallelism. `paper_1804_04512_b200.fastnn` mirrors the reference's host API on top.
"""
from . import configs  # noqa: F401

__all__ = ["configs", "fastnn", "build"]
