"""The reference (fastnn) and the B200 build side by side through their C++ APIs
(tests/cpp/drop_in_parity.cpp; include/b200nn.hpp is the drop-in): MLP, MNIST CNN, CIFAR CNN
3-step training, RBM CD-1, CRBM CD-1, and fit + save_network driven by identical fastnn::Tensor inputs and std::mt19937 streams."""
import subprocess
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu
BIN = Path(__file__).resolve().parents[1] / "oracle" / "_ref" / "drop_in_parity"


@pytest.mark.skipif(not BIN.exists(), reason="drop_in_parity is built where /root/reference exists")
def test_cpp_drop_in_parity(gpu):
    r = subprocess.run([str(BIN)], capture_output=True, text=True, timeout=600)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
    assert r.stdout.count("PASS") == 8
