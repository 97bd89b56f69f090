"""The C ABI (include/b200nn.h): the library builds for sm_100a, loads, exports every declared
symbol, and fails loudly (a CUDA status, never a CPU fallback) when no GPU is present."""
import re
from pathlib import Path

import pytest

from paper_1804_04512_b200 import _lib

ROOT = Path(__file__).resolve().parents[1]


def declared_symbols():
    text = (ROOT / "include" / "b200nn.h").read_text()
    return sorted(set(re.findall(r"\b(b2n_[a-z0-9_]+)\s*\(", text)))


def test_header_matches_binding():
    assert declared_symbols() == sorted(_lib.EXPORTED)


def test_library_exports_every_symbol():
    lib = _lib.load()
    for name in declared_symbols():
        assert hasattr(lib, name), name


def test_library_is_sm100a():
    import subprocess
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", str(_lib.lib_path())], capture_output=True,
                         text=True)
    assert "sm_100a" in out.stdout
    sass = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "-sass", str(_lib.lib_path())], capture_output=True,
                          text=True).stdout
    assert "UTCHMMA" in sass and "UTMALDG" in sass and "LDTM" in sass  # tcgen05.mma, TMA, tcgen05.ld


def test_status_codes_and_no_fallback():
    import torch
    from paper_1804_04512_b200 import configs as CF
    from paper_1804_04512_b200 import fastnn as F
    assert _lib.load().b2n_version() >= 1
    with pytest.raises(F.SpecError):  # spec validation (build_network, network.hpp:285) before any device work
        F.build_network({"input": [784], "layers": []})
    with pytest.raises(F.SpecError):
        F.build_network({"input": [6, 6, 6], "layers": [CF.dense(216, 10), CF.relu(), CF.softmax(), CF.dense(4, 4)]})
    if not torch.cuda.is_available():
        with pytest.raises(F.CudaError):  # no GPU: a CUDA error, not a CPU path
            F.build_network(CF.mlp_spec())
