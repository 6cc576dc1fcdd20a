#!/usr/bin/env python
"""One f4 case (4096 x 4096 Particle7) copied a few times, for ncu captures:
    python tools/f4_one.py SRC_KIND SRC_LIN DST_KIND DST_LIN [knob=value ...]
e.g. python tools/f4_one.py soa_mb col soa_mb row jit_lanes=3"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2106_04284_b200 as llama  # noqa: E402
import workloads as W  # noqa: E402

sk, sl, dk, dl = sys.argv[1:5]
knobs = {k: int(v) for k, v in (a.split("=") for a in sys.argv[5:])}
EXT = [4096, 4096]
sm = llama.Mapping.from_spec(W.PARTICLE7, EXT, (sk, 1, False), lin=sl)
dm = llama.Mapping.from_spec(W.PARTICLE7, EXT, (dk, 1, False), lin=dl)
sb, db = sm.alloc(), dm.alloc()
llama.generate(sm, sb, 1)
print(llama.plan(sm, dm, knobs=knobs))
for _ in range(3):
    llama.copy(sm, sb, dm, db, knobs=knobs)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(5):
    llama.copy(sm, sb, dm, db, knobs=knobs)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 5
print(f"{sk}/{sl} -> {dk}/{dl} {knobs} {(sm.footprint() + dm.footprint()) / ms / 1e6:.0f} GB/s", flush=True)
