#!/usr/bin/env python
"""One transposing copy of a 2-d view pair, repeated (ncu driver for the wide
kernel): wide_once.py SCHEMA EXTENT SRC/LIN DST/LIN [knob=v,...]."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2106_04284_b200 as llama  # noqa: E402
import workloads as W  # noqa: E402

schema, e = W.SCHEMAS[sys.argv[1]], int(sys.argv[2])
(a, sl), (b, dl) = sys.argv[3].split("/"), sys.argv[4].split("/")
knobs = dict((k, int(v)) for k, v in (x.split("=") for x in sys.argv[5].split(","))) if len(sys.argv) > 5 else None
sm = llama.Mapping.from_spec(schema, [e, e], W.resolve_spec(a), lin=sl)
dm = llama.Mapping.from_spec(schema, [e, e], W.resolve_spec(b), lin=dl)
src, dst = sm.alloc(), dm.alloc()
llama.generate(sm, src, 3)
print(llama.plan(sm, dm, knobs=knobs))
for _ in range(3):
    llama.copy(sm, src, dm, dst, knobs=knobs)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(10):
    llama.copy(sm, src, dm, dst, knobs=knobs)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 10
print(f"{a}/{sl} -> {b}/{dl}: {ms:.4f} ms, {(sm.footprint() + dm.footprint()) / ms / 1e6:.0f} GB/s")
