#!/usr/bin/env python
"""Concurrent pinned H2D + D2H throughput (the ceiling for a staged host relayout)."""
import torch
n = 512 << 20
h1 = torch.empty(n, dtype=torch.uint8).pin_memory(); h2 = torch.empty(n, dtype=torch.uint8).pin_memory()
d1 = torch.empty(n, dtype=torch.uint8, device="cuda"); d2 = torch.empty(n, dtype=torch.uint8, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
for _ in range(2):
    with torch.cuda.stream(s1): d1.copy_(h1, non_blocking=True)
    with torch.cuda.stream(s2): h2.copy_(d2, non_blocking=True)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
s1.wait_event(e0); s2.wait_event(e0)
for _ in range(4):
    with torch.cuda.stream(s1): d1.copy_(h1, non_blocking=True)
    with torch.cuda.stream(s2): h2.copy_(d2, non_blocking=True)
ev1, ev2 = torch.cuda.Event(), torch.cuda.Event()
ev1.record(s1); ev2.record(s2)
torch.cuda.current_stream().wait_event(ev1); torch.cuda.current_stream().wait_event(ev2)
e1.record(); torch.cuda.synchronize()
ms = e0.elapsed_time(e1)
print(f"concurrent H2D+D2H: {2 * 4 * n / ms / 1e6:.1f} GB/s total ({4 * n / ms / 1e6:.1f} each way)")
