"""Pinned host -> device copy rate on this box (the e2e path's link), 1 GiB x 5."""
import time

import torch

n = 1 << 30
h = torch.empty(n, dtype=torch.uint8, pin_memory=True)
d = torch.empty(n, dtype=torch.uint8, device="cuda")
s = torch.cuda.Stream()
for _ in range(2):
    with torch.cuda.stream(s):
        d.copy_(h, non_blocking=True)
    s.synchronize()
ts = []
for _ in range(5):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(s):
        e0.record(s)
        d.copy_(h, non_blocking=True)
        e1.record(s)
    s.synchronize()
    ts.append(e0.elapsed_time(e1))
print(f"H2D pinned: {n / (min(ts) / 1e3) / 1e9:.1f} GB/s (best of 5, 1 GiB), times ms {[round(t, 2) for t in ts]}")
