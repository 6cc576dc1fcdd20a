#!/usr/bin/env python
"""One transposing copy (SoA MB column-major -> row-major, 4096 x 4096 Particle7) for ncu."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2106_04284_b200 as llama  # noqa: E402
import workloads as W  # noqa: E402

ext = [4096, 4096]
a = (sys.argv[1] if len(sys.argv) > 1 else "soa_mb")
sm = llama.Mapping.from_spec(W.PARTICLE7, ext, W.resolve_spec(a), lin="col")
dm = llama.Mapping.from_spec(W.PARTICLE7, ext, W.resolve_spec(a), lin="row")
sb, db = sm.alloc(), dm.alloc()
llama.generate(sm, sb, 1)
for _ in range(2):
    llama.copy(sm, sb, dm, db)
torch.cuda.synchronize()
print(llama.plan(sm, dm))
