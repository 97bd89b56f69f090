"""save_network / load_network (network.hpp:552-607) on the device-resident net: the FNN1 bytes the
library writes equal the reference's own save_network output byte for byte (tests/golden/*.fnn1,
make_golden.py checkpoint), a reference checkpoint loads into bit-identical parameters, malformed
files fail with the reference's error type and text, and the `.state` sidecar gives an exact
resume (same subsequent steps as an uninterrupted run)."""
import json
from pathlib import Path

import numpy as np
import pytest

from oracle import oracle as O

pytestmark = pytest.mark.gpu
GOLD = Path(__file__).resolve().parent / "golden"
META = json.loads((GOLD / "meta.json").read_text())
NAMES = ["mlp_small", "mnist_cnn_small", "cifar_cnn_small"]


def net_from_golden(name):
    """the small net with the reference's post-two-step parameters (bitwise, from the golden npz)"""
    from paper_1804_04512_b200 import fastnn as F
    g = np.load(GOLD / f"{name}.npz")
    net = F.build_network(META[name]["spec"])
    orc = O.Net(META[name]["spec"])
    for _ in range(2):
        orc.train_minibatch(g["x"], g["labels"])
    for i in range(net.num_params()):
        net.set_param(i, orc.get(i))
    return net, orc


@pytest.mark.parametrize("name", NAMES)
def test_save_bytes_equal_reference(gpu, name, tmp_path):
    from paper_1804_04512_b200 import fastnn as F
    net, _ = net_from_golden(name)
    p = tmp_path / "n.fnn1"
    F.save_network(net, p)
    assert p.read_bytes() == (GOLD / f"{name}.fnn1").read_bytes()


@pytest.mark.parametrize("name", NAMES)
def test_load_reference_checkpoint(gpu, name):
    from paper_1804_04512_b200 import fastnn as F
    net = F.build_network(META[name]["spec"])
    _, orc = net_from_golden(name)
    F.load_network(net, GOLD / f"{name}.fnn1")
    for i in range(net.num_params()):
        assert np.array_equal(net.get_param(i).ravel().view(np.uint32), orc.get(i).view(np.uint32)), i


@pytest.mark.parametrize("name", NAMES)
def test_malformed_checkpoints(gpu, name, tmp_path):
    from paper_1804_04512_b200 import fastnn as F
    errs = json.loads((GOLD / "checkpoint_errors.json").read_text())
    data = (GOLD / f"{name}.fnn1").read_bytes()
    cases = {"bad_magic": (b"FNN2" + data[4:], F.FormatError), "truncated": (data[:-3], F.LengthError),
             "empty": (b"", F.LengthError),
             "layer_count": (data[:4] + (99).to_bytes(4, "little") + data[8:], F.FormatError),
             "tag": (data[:12] + b"x" + data[13:], F.FormatError)}
    net = F.build_network(META[name]["spec"])
    before = net.params()
    for case, (blob, exc) in cases.items():
        p = tmp_path / f"{case}.fnn1"
        p.write_bytes(blob)
        with pytest.raises(exc) as ei:
            F.load_network(net, p)
        assert str(ei.value) == errs[f"{name}:{case}"], case
    with pytest.raises(F.DataMissingError) as ei:
        F.load_network(net, tmp_path / "_does_not_exist.fnn1")
    assert str(ei.value).startswith("load_network: cannot open ")
    for a, b in zip(before, net.params()):  # a failed load leaves the parameters untouched
        assert np.array_equal(a, b)


def test_resume_with_state(gpu, tmp_path):
    """train 2 steps, checkpoint with state, train 2 more; a fresh net loaded from the checkpoint
    and trained 2 steps lands on the same parameters bit for bit"""
    from paper_1804_04512_b200 import configs as CF, fastnn as F
    spec = CF.NET_CONFIGS["mnist_cnn"](100)
    x = O.uniform_f32(3, 100 * 784).reshape(100, 1, 28, 28)
    lab = O.uniform_int(4, 0, 9, 100)
    a = F.build_network(spec)
    for _ in range(2):
        F.train_minibatch_labels(a, x, lab)
    F.save_network(a, tmp_path / "c.fnn1", with_state=True)
    la = [F.train_minibatch_labels(a, x, lab) for _ in range(2)]
    b = F.build_network(dict(spec, lr=0.5))  # hyper-parameters come back from the sidecar
    F.load_network(b, tmp_path / "c.fnn1", with_state=True)
    lb = [F.train_minibatch_labels(b, x, lab) for _ in range(2)]
    assert la == lb
    for i in range(a.num_params()):
        assert np.array_equal(a.get_param(i), b.get_param(i))
        assert np.array_equal(a.get_param(i, F.VELOCITY), b.get_param(i, F.VELOCITY))
