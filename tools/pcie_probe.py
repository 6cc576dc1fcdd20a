#!/usr/bin/env python
"""Host<->device copy ceiling on this box: pinned H2D alone, D2H alone, and
both at once on two streams (the staged end-to-end copy's ceiling)."""
import torch

n = 1 << 30
h_src = torch.empty(n, dtype=torch.uint8, pin_memory=True)
h_dst = torch.empty(n, dtype=torch.uint8, pin_memory=True)
d_a = torch.empty(n, dtype=torch.uint8, device="cuda")
d_b = torch.empty(n, dtype=torch.uint8, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def timed(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def both():
    cur = torch.cuda.current_stream()
    s1.wait_stream(cur)
    s2.wait_stream(cur)
    with torch.cuda.stream(s1):
        d_a.copy_(h_src, non_blocking=True)
    with torch.cuda.stream(s2):
        h_dst.copy_(d_b, non_blocking=True)
    cur.wait_stream(s1)
    cur.wait_stream(s2)


ms = timed(lambda: d_a.copy_(h_src, non_blocking=True))
print(f"H2D alone     {n / ms / 1e6:.1f} GB/s")
ms = timed(lambda: h_dst.copy_(d_b, non_blocking=True))
print(f"D2H alone     {n / ms / 1e6:.1f} GB/s")
ms = timed(both)
print(f"H2D + D2H     {2 * n / ms / 1e6:.1f} GB/s total ({n / ms / 1e6:.1f} each way)")
