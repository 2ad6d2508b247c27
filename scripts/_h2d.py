import torch, time
n, od, sb = 16384, 27648, 980704
h = torch.empty(n * od, dtype=torch.uint8).pin_memory()
d = torch.empty(n * od, dtype=torch.uint8, device="cuda")
reg = torch.empty(n * sb, dtype=torch.uint8, device="cuda")
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for _ in range(2): d.copy_(h, non_blocking=True)
torch.cuda.synchronize()
e0.record()
for _ in range(10): d.copy_(h, non_blocking=True)
e1.record(); torch.cuda.synchronize()
print("contiguous H2D GB/s", 10 * n * od / (e0.elapsed_time(e1) * 1e-3) / 1e9)
dst = reg.view(n, sb)[:, 64:64 + od]
for _ in range(2): dst.copy_(h.view(n, od), non_blocking=True)
torch.cuda.synchronize()
e0.record()
for _ in range(10): dst.copy_(h.view(n, od), non_blocking=True)
e1.record(); torch.cuda.synchronize()
print("2D H2D GB/s", 10 * n * od / (e0.elapsed_time(e1) * 1e-3) / 1e9)
