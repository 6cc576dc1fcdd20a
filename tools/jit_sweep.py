#!/usr/bin/env python
"""Sweeps the JIT permute's geometry knobs (jit_tile, jit_stages,
jit_dst_bufs) on chosen C3 pairs; prints GB/s per setting.
    python tools/jit_sweep.py [--records N] [--pairs a:b,...]"""
import argparse
import itertools
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2106_04284_b200 as llama  # noqa: E402
import workloads as W  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--records", type=int, default=1 << 24)
ap.add_argument("--pairs", default="soa_mb:aos,soa_mb:aos_aligned,aos:soa_mb,aos_aligned:soa_mb,aos:aos_aligned,aos_aligned:aos")
ap.add_argument("--iters", type=int, default=5)
ap.add_argument("--extra", default="", help="knobs added to every setting, k=v,...")
a = ap.parse_args()
extra = {k: int(v) for k, v in (kv.split("=") for kv in a.extra.split(",") if kv)}
n = a.records
views = {}
for pair in a.pairs.split(","):
    s, d = pair.split(":")
    for k in (s, d):
        if k not in views:
            m = llama.Mapping(W.HEP100, [n], *W.MAPPINGS[k])
            views[k] = (m, m.alloc(), m.alloc())
            llama.generate(m, views[k][1], 42)
grid = {"jit_tile": [32, 64, 128], "jit_stages": [2, 3, 4], "jit_dst_bufs": [2, 3]}
for pair in a.pairs.split(","):
    s, d = pair.split(":")
    sm, sb, _ = views[s]
    dm, _, db = views[d]
    res = []
    for vals in itertools.product(*grid.values()):
        knobs = dict(zip(grid.keys(), vals), jit=2, **extra)
        try:
            pl = llama.plan(sm, dm, path="permute", knobs=knobs)
        except llama.LlamaError:
            continue
        if not pl["jit"]:
            continue
        if pl["tile_records"] != knobs["jit_tile"]:
            continue
        llama.copy(sm, sb, dm, db, path="permute", knobs=knobs)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(a.iters):
            llama.copy(sm, sb, dm, db, path="permute", knobs=knobs)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / a.iters
        gbs = (sm.footprint() + dm.footprint()) / ms / 1e6
        res.append((gbs, knobs, pl["smem_bytes"]))
        print(f"{s:>12} -> {d:<12} {knobs} smem={pl['smem_bytes']} {gbs:.0f} GB/s", flush=True)
    res.sort(key=lambda x: -x[0])
    print(f"BEST {s} -> {d}: {res[0] if res else None}", flush=True)
