import torch, time
x = torch.empty(369_360_896 // 4, dtype=torch.float32).pin_memory()
y = torch.empty_like(x, device="cuda")
for _ in range(3): y.copy_(x, non_blocking=True)
torch.cuda.synchronize()
s = torch.cuda.Event(enable_timing=True); e = torch.cuda.Event(enable_timing=True)
s.record(); 
for _ in range(5): y.copy_(x, non_blocking=True)
e.record(); torch.cuda.synchronize()
ms = s.elapsed_time(e) / 5
print(f"H2D 369 MB pinned: {ms:.3f} ms = {369.36/ms:.1f} GB/s")
z = torch.empty(65536, dtype=torch.float32).pin_memory(); zz = torch.empty(65536, device="cuda")
s.record()
for _ in range(100): z.copy_(zz, non_blocking=True)
e.record(); torch.cuda.synchronize(); print(f"D2H 256 KB: {s.elapsed_time(e)/100*1000:.1f} us")
