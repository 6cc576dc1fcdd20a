#!/usr/bin/env python
"""Default plans of transposing copies (rank-2 views, different storage
orders) over kinds x storage-order pairs: worst first."""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2106_04284_b200 as llama  # noqa: E402
import workloads as W  # noqa: E402

PEAK = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]
KINDS = ["aos", "aos_aligned", "soa_mb", "soa_sb", "aosoa8"]
LINS = [("row", "col"), ("col", "row"), ("row", "morton"), ("morton", "row"), ("col", "morton")]
rows = []
SIZES = {"particle7": 4096, "listing1": 4096, "hep100": 1024}
KN = dict((k, int(v)) for k, v in (x.split("=") for x in sys.argv[2].split(","))) if len(sys.argv) > 2 else None
for schema in (sys.argv[1].split(",") if len(sys.argv) > 1 else list(SIZES)):
    e = SIZES[schema]
    sch = W.SCHEMAS[schema]
    warm = None
    for sl, dl in LINS:
        maps_s = {k: llama.Mapping.from_spec(sch, [e, e], W.resolve_spec(k), lin=sl) for k in KINDS}
        maps_d = {k: llama.Mapping.from_spec(sch, [e, e], W.resolve_spec(k), lin=dl) for k in KINDS}
        src = {k: m.alloc() for k, m in maps_s.items()}
        dst = {k: m.alloc() for k, m in maps_d.items()}
        for k, m in maps_s.items():
            llama.generate(m, src[k], 3)
        if warm is None:
            t = time.time() + 0.3
            while time.time() < t:
                llama.copy(maps_s["aos"], src["aos"], maps_d["soa_mb"], dst["soa_mb"])
                torch.cuda.synchronize()
            warm = True
        for a in KINDS:
            for b in KINDS:
                sm, dm = maps_s[a], maps_d[b]
                llama.copy(sm, src[a], dm, dst[b], knobs=KN)
                torch.cuda.synchronize()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                for _ in range(5):
                    llama.copy(sm, src[a], dm, dst[b], knobs=KN)
                e1.record()
                torch.cuda.synchronize()
                ms = e0.elapsed_time(e1) / 5
                g = (sm.footprint() + dm.footprint()) / ms / 1e6
                pl = llama.plan(sm, dm, knobs=KN)
                rows.append((g / PEAK, g, schema, e, f"{a}/{sl}", f"{b}/{dl}", pl["path"],
                             " jit" if pl["jit"] else " wide" if pl["wide"] else ""))
        del src, dst
        torch.cuda.empty_cache()
rows.sort()
for f, g, schema, e, a, b, path, jit in rows:
    print(f"{f:6.3f} {g:7.0f} GB/s  {schema:9s} {e}x{e}  {a:>18s} -> {b:<18s} {path}{jit}")
