import os
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs the CUDA library)")


def norm_err(got, want) -> float:
    """SURVEY 8(d) parity metric: ||got - want||_inf / ||want||_inf."""
    got = np.asarray(got, np.float64)
    want = np.asarray(want, np.float64)
    den = np.abs(want).max()
    return float(np.abs(got - want).max() / (den if den > 0 else 1.0))


def rel_err(a, b) -> float:
    """oracles.hpp:27: |a-b| / max(1, |b|), worst element."""
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    return float((np.abs(a - b) / np.maximum(1.0, np.abs(b))).max())


@pytest.fixture(scope="session")
def gpu():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch.device("cuda:0")


def check_argmax(am, probs_gpu, probs_ref, am_ref, max_near_frac=0.01):
    """Prediction argmax contract (network.hpp:66-72, first maximum wins): bit-exact on every row
    whose top-2 reference probabilities are separated by more than twice the measured probability
    error; on the remaining near-tied rows the GPU's pick must be one of the tied classes. Returns the
    number of near-tied rows, which is bounded (<= max_near_frac of the rows, at least 1 allowed)."""
    am = np.asarray(am).ravel()
    am_ref = np.asarray(am_ref).ravel()
    pg = np.asarray(probs_gpu, np.float64).reshape(am.size, -1)
    pr = np.asarray(probs_ref, np.float64).reshape(am.size, -1)
    err = float(np.abs(pg - pr).max())
    top2 = np.sort(pr, axis=1)[:, -2:]
    band = 2.0 * err + 1e-12
    near = (top2[:, 1] - top2[:, 0]) <= band
    assert np.array_equal(am[~near], am_ref[~near]), "argmax differs outside the near-tie band"
    rows = np.nonzero(near)[0]
    assert np.all(pr[rows, am[rows]] >= top2[rows, 1] - band), "near-tie pick is not one of the tied classes"
    n = int(near.sum())
    assert n <= max(1, int(max_near_frac * am.size)), (n, am.size)
    print(f"argmax: {am.size - n}/{am.size} rows bit-exact, {n} near-tied within 2x max|dp| = {band:.2e}, "
          f"{int((am[near] != am_ref[near]).sum())} of them picked differently")
    return n
