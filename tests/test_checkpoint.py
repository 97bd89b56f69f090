"""The FNN1 checkpoint fixtures (tests/golden/*.fnn1, written by the reference's save_network,
network.hpp:552-573) parsed by a plain reader of the documented layout hold exactly the golden
post-step parameters and the reference's node tags (incl. the implicit flatten before a dense
layer, network.hpp:309-312). Pins the byte fixtures the GPU checkpoint tests compare against."""
import json
import struct
from pathlib import Path

import numpy as np
import pytest

GOLD = Path(__file__).resolve().parent / "golden"
TAGS = {"mlp_small": ["dense", "sigmoid", "dense", "sigmoid", "dense", "softmax"],
        "mnist_cnn_small": ["conv", "sigmoid", "maxpool", "conv", "sigmoid", "maxpool", "flatten", "dense", "sigmoid",
                            "dense", "softmax"],
        "cifar_cnn_small": ["conv", "relu", "maxpool", "conv", "relu", "maxpool", "flatten", "dense", "relu", "dense",
                            "softmax"]}


def read_fnn1(blob: bytes):
    pos = 0

    def take(n):
        nonlocal pos
        assert pos + n <= len(blob), "truncated"
        pos += n
        return blob[pos - n:pos]

    assert take(4) == b"FNN1"
    layers = []
    for _ in range(struct.unpack("<I", take(4))[0]):
        tag = take(struct.unpack("<I", take(4))[0]).decode()
        tensors = []
        for _ in range(struct.unpack("<I", take(4))[0]):
            rank = struct.unpack("<I", take(4))[0]
            dims = struct.unpack(f"<{rank}Q", take(8 * rank))
            n = int(np.prod(dims))
            tensors.append(np.frombuffer(take(4 * n), "<f4").reshape(dims))
        layers.append((tag, tensors))
    assert pos == len(blob)
    return layers


@pytest.mark.parametrize("name", list(TAGS))
def test_golden_checkpoint_layout(name):
    g = np.load(GOLD / f"{name}.npz")
    layers = read_fnn1((GOLD / f"{name}.fnn1").read_bytes())
    assert [t for t, _ in layers] == TAGS[name]
    flat = [t for _, ts in layers for t in ts]
    assert len(flat) == len([k for k in g.files if k.startswith("final")])
    for i, t in enumerate(flat):
        assert np.array_equal(t.ravel().view(np.uint32), g[f"final{i}"].view(np.uint32)), i


def test_error_texts_recorded():
    errs = json.loads((GOLD / "checkpoint_errors.json").read_text())
    assert errs["mlp_small:bad_magic"] == "load_network: bad magic; expected FNN1"
    assert errs["mnist_cnn_small:layer_count"] == "load_network: checkpoint has 99 layers; network has 11"
