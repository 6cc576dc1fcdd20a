#!/usr/bin/env python
"""Probe: HEP100 transposing copies through the JIT transpose with 4- / 8-row
tiles (knob jit_tile) against the wide kernel: parity with the oracle at
256 x 256, GB/s at 1024 x 1024."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle  # noqa: E402
import paper_2106_04284_b200 as llama  # noqa: E402
import workloads as W  # noqa: E402

PEAK = 6550.0
PAIRS = [tuple(x.split(":")) for x in sys.argv[1].split(",")] if len(sys.argv) > 1 else [
    ("aos", "col", "soa_mb", "row"), ("aos", "row", "aos", "col"), ("aos", "row", "aos_aligned", "col"),
    ("aos_aligned", "col", "soa_sb", "row"), ("aos_aligned", "col", "aos", "row"), ("soa_mb", "col", "aos", "row"),
    ("aos", "col", "soa_sb", "row"), ("aos_aligned", "row", "aos_aligned", "col")]
KNOBS = [None] + [dict((k, int(v)) for k, v in (kv.split("=") for kv in ks.split("+"))) for ks in sys.argv[2].split(",")] \
    if len(sys.argv) > 2 else [None, {"jit_tile": 128}, {"jit_tile": 256}]
for a, sl, b, dl in PAIRS:
    for kn in KNOBS:
        try:
            e = 256
            sm = llama.Mapping.from_spec(W.HEP100, [e, e], W.resolve_spec(a), lin=sl)
            dm = llama.Mapping.from_spec(W.HEP100, [e, e], W.resolve_spec(b), lin=dl)
            pl = llama.plan(sm, dm, knobs=kn)
            so = oracle.mapping_from_spec(W.HEP100, [e, e], W.resolve_spec(a), lin=sl)
            do = oracle.mapping_from_spec(W.HEP100, [e, e], W.resolve_spec(b), lin=dl)
            sb = sm.alloc()
            llama.generate(sm, sb, 5, pad_byte=0xCD)
            exp = oracle.copy(so, oracle.make_view(so, 5, pad_fill=0xCD), do, nthreads=8)
            db = dm.alloc()
            for t in db:
                t.fill_(0x5A)
            llama.copy(sm, sb, dm, db, knobs=kn)
            torch.cuda.synchronize()
            ok = all(np.array_equal(t.cpu().numpy(), exp[j]) for j, t in enumerate(db))
            e = 1024
            sm = llama.Mapping.from_spec(W.HEP100, [e, e], W.resolve_spec(a), lin=sl)
            dm = llama.Mapping.from_spec(W.HEP100, [e, e], W.resolve_spec(b), lin=dl)
            sb, db = sm.alloc(), dm.alloc()
            for _ in range(3):
                llama.copy(sm, sb, dm, db, knobs=kn)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(10):
                llama.copy(sm, sb, dm, db, knobs=kn)
            e1.record()
            torch.cuda.synchronize()
            g = (sm.footprint() + dm.footprint()) / (e0.elapsed_time(e1) / 10) / 1e6
            print(f"{a}/{sl} -> {b}/{dl} {kn}: {'jit' if pl['jit'] else 'wide' if pl['wide'] else pl['path']} "
                  f"T={pl['tile_records']} smem={pl['smem_bytes']} parity={ok} {g:.0f} GB/s {g / PEAK:.3f}", flush=True)
        except Exception as ex:  # noqa: BLE001
            print(f"{a}/{sl} -> {b}/{dl} {kn}: ERROR {ex}", flush=True)
