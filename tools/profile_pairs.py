#!/usr/bin/env python
"""Runs selected mapping pairs of a BASELINE config a few times (for ncu
captures and quick timing).  Usage:
    python tools/profile_pairs.py --config C2 --pairs aos:soa_mb,aosoa8:soa_mb --iters 3 [--path permute]
        [--knobs stages=3,dst_bufs=2]   (llama_knob overrides, paper_2106_04284_b200.KNOBS)
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
if os.environ.get("LLAMA_PKG_ROOT"):  # A/B against another build of the package
    sys.path.insert(0, os.environ["LLAMA_PKG_ROOT"])
import torch  # noqa: E402

import paper_2106_04284_b200 as llama  # noqa: E402
import workloads as W  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="C2")
ap.add_argument("--pairs", default="aos:soa_mb")
ap.add_argument("--iters", type=int, default=3)
ap.add_argument("--path", default=None)
ap.add_argument("--tile", type=int, default=0)
ap.add_argument("--records", type=int, default=0)
ap.add_argument("--knobs", default="")
ap.add_argument("--subcfg", default="", help="schema and extents of a bench sub-config (bench.SUBCFG); views may be kind/lin")
ap.add_argument("--stagger", type=int, default=0, help="allocate blob k at a k * STAGGER byte offset (alignment study)")
ap.add_argument("--pool", action="store_true", help="all blobs of a side in one allocation, back to back")
a = ap.parse_args()
knobs = {k: int(v) for k, v in (kv.split("=") for kv in a.knobs.split(",") if kv)} or None
if a.subcfg:
    import bench
    cfg = bench.SUBCFG[a.subcfg]
else:
    cfg = W.CONFIGS[a.config]
schema = W.SCHEMAS[cfg["schema"]]
ext = [a.records] if a.records else list(cfg["extents"])


def view(spec):
    kind, _, lin = spec.partition("/")
    return llama.Mapping.from_spec(schema, ext, W.resolve_spec(kind), lin=lin or "row")
warmed = False
for pair in a.pairs.split(","):
    s, d = pair.split(":")
    sm, dm = view(s), view(d)
    def alloc(m):
        if a.pool:
            sizes = [(x + 255) // 256 * 256 for x in m.blob_sizes()]
            base = torch.empty(sum(sizes) + 256, dtype=torch.uint8, device="cuda")
            out, o = [], 0
            for x, sz in zip(m.blob_sizes(), sizes):
                out.append(base[o:o + x])
                o += sz
            return out
        if not a.stagger:
            return m.alloc()
        return [torch.empty(x + k * a.stagger + 16, dtype=torch.uint8, device="cuda")[k * a.stagger:k * a.stagger + x]
                for k, x in enumerate(m.blob_sizes())]
    sb, db = alloc(sm), alloc(dm)
    llama.generate(sm, sb, 42)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    llama.copy(sm, sb, dm, db, path=a.path, tile_records=a.tile, knobs=knobs)
    if not warmed:  # bring the GPU to its load clocks before the first timed pair (~200 ms of copies)
        import time
        t_end = time.time() + 0.2
        while time.time() < t_end:
            llama.copy(sm, sb, dm, db, path=a.path, tile_records=a.tile, knobs=knobs)
            torch.cuda.synchronize()
        warmed = True
    e0.record()
    for _ in range(a.iters):
        llama.copy(sm, sb, dm, db, path=a.path, tile_records=a.tile, knobs=knobs)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / a.iters
    nbytes = sm.footprint() + dm.footprint()
    print(f"{s:>12} -> {d:<12} {llama.plan(sm, dm, path=a.path, tile_records=a.tile, knobs=knobs)} {ms:.3f} ms "
          f"{nbytes / ms / 1e6:.0f} GB/s", flush=True)
    del sb, db
