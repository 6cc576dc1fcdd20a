#!/usr/bin/env python
"""Knob sweep of the JIT transposing copy (llb_jit_transpose) on the f4 cases
(4096 x 4096 Particle7): GB/s per knob set (block / per-record programs,
block orders, tile, stages / buffers)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2106_04284_b200 as llama  # noqa: E402
import workloads as W  # noqa: E402

EXT = [4096, 4096]
AOS, SOA = ("aos", 1, False), ("soa_mb", 1, False)
CASES = [(AOS, "row", AOS, "col"), (AOS, "row", SOA, "col"), (SOA, "col", SOA, "row"), (AOS, "row", AOS, "morton"),
         (SOA, "morton", AOS, "col"), (SOA, "row", AOS, "col")]
KNOBS = [{}, {"jit_block": 0}, {"jit_bmap": 0}, {"jit_bmap": 1}, {"jit_bmap": 2}, {"jit_bmap": 3}, {"jit_bmap": 4},
         {"jit_tile": 1024}, {"jit_tile": 512}, {"jit_stages": 2, "jit_dst_bufs": 2}, {"jit_stages": 3, "jit_dst_bufs": 3},
         {"jit": 0}]
if len(sys.argv) > 1:  # knob sets as JSON: python tools/f4_sweep.py '[{}, {"jit_block": 0}]'
    import json
    KNOBS = json.loads(sys.argv[1])
for sspec, slin, dspec, dlin in CASES:
    sm = llama.Mapping.from_spec(W.PARTICLE7, EXT, sspec, lin=slin)
    dm = llama.Mapping.from_spec(W.PARTICLE7, EXT, dspec, lin=dlin)
    sb, db = sm.alloc(), dm.alloc()
    llama.generate(sm, sb, 1)
    for knobs in KNOBS:
        pl = llama.plan(sm, dm, knobs=knobs)
        llama.copy(sm, sb, dm, db, knobs=knobs)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(5):
            llama.copy(sm, sb, dm, db, knobs=knobs)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 5
        print(f"{sspec[0]}/{slin} -> {dspec[0]}/{dlin} {knobs} jit={pl['jit']} smem={pl['smem_bytes']} "
              f"{(sm.footprint() + dm.footprint()) / ms / 1e6:.0f} GB/s", flush=True)
