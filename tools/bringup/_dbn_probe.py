"""probe: dbn_pretrain throughput on the MNIST-shape 784-500 first layer (60000 rows, batch 100),
C++-style uniform source (Python Mt19937 callback) -- where the time goes"""
import time

import numpy as np

from paper_1804_04512_b200 import fastnn as F

rng = np.random.default_rng(1)
data = (rng.random((60000, 784)) < 0.3).astype(np.float32)
r = F.Rbm(500, 784)
r.init(42)
F.dbn_pretrain([r], data[:1000], 1, 0.1, 100, F.Mt19937(5))  # plans / graphs
for n in (60000,):
    t0 = time.perf_counter()
    rep = F.dbn_pretrain([r], data[:n], 1, 0.1, 100, F.Mt19937(5))
    dt = time.perf_counter() - t0
    print(f"dbn 784-500 1 epoch n={n}: {dt*1e3:.1f} ms, {n/dt:.0f} samples/s, recon {rep.recon[0][0]:.3f}")
m = F.Mt19937(5)
t0 = time.perf_counter()
for _ in range(600):
    m.canonical(50000)
dt = time.perf_counter() - t0
print(f"host Mt19937.canonical(50000) x600: {dt*1e3:.1f} ms ({dt/600*1e6:.1f} us/step)")
