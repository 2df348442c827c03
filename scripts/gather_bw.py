#!/usr/bin/env python3
"""Microbenchmark: random 128-byte row gather vs streaming copy (torch kernels)."""
import torch

R = 3_000_000
src = torch.randn(R, 32, device="cuda")
dst = torch.empty_like(src)
perm = torch.randperm(R, device="cuda")
sorted_idx = torch.arange(R, device="cuda")


def bench(f, reps=20):
    for _ in range(3):
        f()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps):
        f()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / reps


nbytes = 2 * R * 128
t = bench(lambda: dst.copy_(src))
print(f"copy        {nbytes / t / 1e6:8.1f} GB/s")
t = bench(lambda: torch.index_select(src, 0, sorted_idx, out=dst))
print(f"gather seq  {nbytes / t / 1e6:8.1f} GB/s")
t = bench(lambda: torch.index_select(src, 0, perm, out=dst))
print(f"gather rand {nbytes / t / 1e6:8.1f} GB/s")
t = bench(lambda: dst.index_copy_(0, perm, src))
print(f"scatter rand {nbytes / t / 1e6:8.1f} GB/s")
