import torch, time
x = torch.empty(100 << 20, dtype=torch.uint8).pin_memory()
d = torch.empty(100 << 20, dtype=torch.uint8, device="cuda")
s = torch.cuda.Stream()
for _ in range(3): d.copy_(x, non_blocking=True)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(); 
for _ in range(10): d.copy_(x, non_blocking=True)
e1.record(); torch.cuda.synchronize()
print("H2D GB/s", 10 * (100 << 20) / (e0.elapsed_time(e1) * 1e-3) / 1e9)
