"""Single-shot K-step timings of the streamed RBM loop as bench.py takes them (fresh device inputs, a short
warm-up call, one timed call) -- with and without an L2 flush / a full-length warm-up over the same buffers."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
from paper_1804_04512_b200 import fastnn as F

B, H, V, K = 100, 500, 784, int(sys.argv[1]) if len(sys.argv) > 1 else 20
r = F.Rbm(H, V)
r.init(1)
dev = torch.device("cuda", 0)
s = torch.cuda.ExternalStream(r.stream_handle())
flush = torch.empty(512 << 18, device=dev)


def timed(fn):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record(s)
    fn()
    e1.record(s)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) * 1e3 / K


for mode in ("bench", "bench+flush", "fullwarm+flush", "bench", "fullwarm+flush"):
    out = []
    for trial in range(5):
        v = (torch.rand(K * B, V, device=dev) < 0.5).float()
        u = torch.rand(K * B, H, device=dev, dtype=torch.float64)
        w = K if mode.startswith("fullwarm") else 5
        r.train_stream_ptr(v.data_ptr(), u.data_ptr(), w, B, 0.1)
        if "flush" in mode:
            flush.zero_()
        out.append(timed(lambda: r.train_stream_ptr(v.data_ptr(), u.data_ptr(), K, B, 0.1)))
    print(f"{mode:16s} K={K}: " + " ".join(f"{x:.1f}" for x in out))
