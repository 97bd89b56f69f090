"""Per-op CUDA-event timings of one config's step (the planner's ops, b2n_*_profile), for tuning.
    python tools/diag/opprof.py imagenet_cnn [steps]"""
import sys
sys.path.insert(0, "/root/repo")
import bench

name = sys.argv[1]
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 10
dist = bench.Dist()
w = bench.make_work(name, dist, 0, None)
for _ in range(3):
    w.step()
tot = 0.0
for op in w.profile(steps):
    tot += op["ms"]
    print(f"{op['name']:32s} {op['ms'] * 1e3:9.1f} us  kernels {op['kernels']}  "
          f"{op['flops'] / max(op['ms'], 1e-9) / 1e9:8.2f} TFLOP/s  {op['bytes'] / max(op['ms'], 1e-9) / 1e6:8.1f} GB/s")
print(f"{'total':32s} {tot * 1e3:9.1f} us")
