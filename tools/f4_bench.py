#!/usr/bin/env python
"""f4 measurements: copies between differently linearised views (a relayout
plus an N-d transpose / Morton reorder) and the cost of Trace / Heatmap
instrumentation, on 16M Particle7 records (4096 x 4096)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
if os.environ.get("LLAMA_PKG_ROOT"):
    sys.path.insert(0, os.environ["LLAMA_PKG_ROOT"])
import torch  # noqa: E402

import paper_2106_04284_b200 as llama  # noqa: E402
import workloads as W  # noqa: E402

EXT = [4096, 4096]
AOS, SOA = ("aos", 1, False), ("soa_mb", 1, False)


def timed(fn, iters=5):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(iters):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / iters


def copy_case(sspec, slin, dspec, dlin, trace=None, path=None):
    sm = llama.Mapping.from_spec(W.PARTICLE7, EXT, sspec, lin=slin)
    dm = llama.Mapping.from_spec(W.PARTICLE7, EXT, dspec, lin=dlin)
    if trace:
        sm, dm = sm.traced(**trace), dm.traced(**trace)
    sb, db = sm.alloc(), dm.alloc()
    llama.generate(sm, sb, 1)
    ms = timed(lambda: llama.copy(sm, sb, dm, db, path=path))
    gb = (sm.footprint() + dm.footprint()) / (ms * 1e6)
    print(f"copy {sspec[0]}/{slin} -> {dspec[0]}/{dlin} trace={trace} path={llama.plan(sm, dm, path=path)['path']}: "
          f"{ms:.3f} ms {gb:.0f} GB/s", flush=True)


def move_case(spec, trace=None):
    n = EXT[0] * EXT[1]
    m = llama.Mapping.from_spec(W.PARTICLE7, [n], spec)
    if trace:
        m = m.traced(**trace)
    b = m.alloc()
    for t in b:
        t.zero_()
    path = llama.nbody_move(m, b, 1e-4)
    ms = timed(lambda: llama.nbody_move(m, b, 1e-4))
    print(f"move {spec[0]} trace={trace} path={path}: {ms:.3f} ms {36 * n / (ms * 1e6):.0f} GB/s useful", flush=True)


copy_case(AOS, "row", SOA, "row")
copy_case(AOS, "row", SOA, "row", path="naive")
copy_case(AOS, "row", AOS, "col")
copy_case(AOS, "row", SOA, "col")
copy_case(SOA, "col", SOA, "row")
copy_case(AOS, "row", AOS, "morton")
copy_case(SOA, "morton", AOS, "col")
copy_case(AOS, "col", SOA, "col")
copy_case(AOS, "row", SOA, "row", trace={"fields": True})
copy_case(AOS, "row", SOA, "row", trace={"fields": True, "bytes": True})
move_case(SOA)
move_case(SOA, trace={"fields": True})
move_case(SOA, trace={"fields": True, "bytes": True})
move_case(AOS, trace={"fields": True})
