import torch, time
n = 276 * 1024 * 1024 // 4
h = torch.empty(n, dtype=torch.float32, pin_memory=True); d = torch.empty(n, dtype=torch.float32, device="cuda")
for _ in range(3): d.copy_(h, non_blocking=True)
torch.cuda.synchronize()
e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
e0.record(); 
for _ in range(10): d.copy_(h, non_blocking=True)
e1.record(); torch.cuda.synchronize()
print("H2D GB/s", 10 * n * 4 / (e0.elapsed_time(e1) / 1e3) / 1e9)
e0.record()
for _ in range(10): h.copy_(d, non_blocking=True)
e1.record(); torch.cuda.synchronize()
print("D2H GB/s", 10 * n * 4 / (e0.elapsed_time(e1) / 1e3) / 1e9)
