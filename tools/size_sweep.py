#!/usr/bin/env python
"""Default plans across sizes: GB/s of representative pairs of every config
family at several record counts / extents (looks for planner cliffs)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2106_04284_b200 as llama  # noqa: E402
import workloads as W  # noqa: E402


def rate(sm, dm, iters=5):
    sb, db = sm.alloc(), dm.alloc()
    llama.generate(sm, sb, 1)
    llama.copy(sm, sb, dm, db)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(iters):
        llama.copy(sm, sb, dm, db)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / iters
    return (sm.footprint() + dm.footprint()) / ms / 1e6, llama.plan(sm, dm)


ONE_D = [("particle7", [("aos", "soa_mb"), ("soa_mb", "aosoa8"), ("aosoa32", "aos")]),
         ("listing1", [("aos", "soa_mb"), ("aos_aligned", "split_pos"), ("aosoa32", "soa_sb")]),
         ("hep100", [("aos", "soa_mb"), ("soa_mb", "aos_aligned"), ("split_hep", "aos")])]
for schema, pairs in ONE_D:
    for n in (1 << 18, 1 << 20, 1 << 22, 1 << 24):
        if schema == "hep100" and n > 1 << 23:
            continue
        for a, b in pairs:
            sm = llama.Mapping.from_spec(W.SCHEMAS[schema], [n], W.resolve_spec(a))
            dm = llama.Mapping.from_spec(W.SCHEMAS[schema], [n], W.resolve_spec(b))
            g, pl = rate(sm, dm)
            print(f"{schema:9s} {n:>9d} {a:>11s} -> {b:<11s} {pl['path']:9s} jit={int(pl['jit'])} T={pl['tile_records']:5d} "
                  f"{g:7.0f} GB/s", flush=True)
for ext in ([512, 512], [1024, 1024], [2048, 4096], [4096, 4096], [8192, 8192]):
    for (sk, sl), (dk, dl) in ((("aos", "row"), ("soa_mb", "col")), (("soa_mb", "col"), ("soa_mb", "row")),
                               (("aos", "row"), ("aos", "col")), (("aos", "row"), ("aos", "morton"))):
        if dl == "morton" and ext[0] != ext[1]:
            continue
        sm = llama.Mapping.from_spec(W.PARTICLE7, ext, (sk, 1, False), lin=sl)
        dm = llama.Mapping.from_spec(W.PARTICLE7, ext, (dk, 1, False), lin=dl)
        g, pl = rate(sm, dm)
        print(f"particle7 {ext[0]}x{ext[1]} {sk}/{sl} -> {dk}/{dl} {pl['path']} jit={int(pl['jit'])} "
              f"T={pl['tile_records']} {g:7.0f} GB/s", flush=True)
