"""dbn_pretrain (energy.hpp:208-240): the oracle's restatement (CD-1 per batch in file order on the
previous layer's hidden means, one mt19937 stream across layers / epochs / batches) pinned
bit-exactly to the reference's own dbn_pretrain (tests/golden/dbn.npz), and the numpy MT19937
stream the Python API draws from equal to std::mt19937 + generate_canonical<double,53>."""
import sys
from pathlib import Path

import numpy as np
import pytest

from oracle import oracle as O

GOLD = Path(__file__).resolve().parent / "golden"
sys.path.insert(0, str(GOLD))
import make_golden as MG  # noqa: E402


def test_oracle_dbn_golden():
    g = np.load(GOLD / "dbn.npz")
    c = MG.DBN_CASE
    stack, data = MG.dbn_case_inputs()
    out, recon = O.dbn_pretrain(stack, data, c["epochs"], c["lr"], c["batch"], c["seed"])
    assert np.array_equal(np.array(recon), g["recon"])
    for l, (W, bv, bh) in enumerate(out):
        for name, a in (("W", W), ("bv", bv), ("bh", bh)):
            assert np.array_equal(a.view(np.uint32), g[f"{name}{l}"].view(np.uint32)), (name, l)


def test_python_uniform_stream_is_std_mt19937():
    from paper_1804_04512_b200.fastnn import Mt19937
    rng = Mt19937(5)
    got = np.concatenate([rng.canonical(7), rng.canonical(1000), rng.canonical(3)])
    assert np.array_equal(got, O.canonical_f64(5, 1010))


@pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built (needs /root/reference)")
def test_oracle_dbn_vs_live_reference_errors():
    stack, data = MG.dbn_case_inputs()
    with pytest.raises(RuntimeError, match="dbn_pretrain: layer 1 expects 20 visible units but layer 0 provides 24"):
        O.ref_dbn_pretrain([stack[0], (stack[1][0][:, :20], stack[1][1][:20], stack[1][2])], data, 1, 0.1, 16, 5)
