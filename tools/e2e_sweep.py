#!/usr/bin/env python
"""End-to-end staged copy (pinned host -> device relayout -> pinned host) for
a few slab sizes: GB/s of (src + dst) bytes, like bench.py's e2e."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2106_04284_b200 as llama
import workloads as W
n = 16_777_216
sm = llama.Mapping(W.PARTICLE7, [n], "aos"); dm = llama.Mapping(W.PARTICLE7, [n], "soa_mb")
hs = [torch.empty(s, dtype=torch.uint8).pin_memory() for s in sm.blob_sizes()]
hd = [torch.empty(s, dtype=torch.uint8).pin_memory() for s in dm.blob_sizes()]
ds = sm.alloc(); llama.generate(sm, ds, 42)
for h, d in zip(hs, ds): h.copy_(d)
nb = sm.footprint() + dm.footprint()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
# plain H2D / D2H rates for context
x = torch.empty(sm.footprint(), dtype=torch.uint8, device="cuda")
e0.record(); x.copy_(hs[0], non_blocking=True); e1.record(); torch.cuda.synchronize()
print(f"H2D pinned {sm.footprint() / e0.elapsed_time(e1) / 1e6:.1f} GB/s")
e0.record(); hs[0].copy_(x, non_blocking=True); e1.record(); torch.cuda.synchronize()
print(f"D2H pinned {sm.footprint() / e0.elapsed_time(e1) / 1e6:.1f} GB/s")
for mb in (8, 16, 32, 64, 128, 256):
    st = llama.Stager(mb << 20)
    llama.copy_staged(st, sm, hs, dm, hd); torch.cuda.synchronize()
    e0.record()
    for _ in range(3):
        llama.copy_staged(st, sm, hs, dm, hd)
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 3
    print(f"slab {mb:4d} MiB: {ms:.1f} ms  {nb / ms / 1e6:.1f} GB/s (src+dst)")
    del st
