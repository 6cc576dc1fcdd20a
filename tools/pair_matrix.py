#!/usr/bin/env python
"""Default plans over every ordered pair of the mapping kinds of a schema
(looks for planner cliffs outside the bench's configs):
    python tools/pair_matrix.py [schema records]...   e.g. particle7 16777216 listing1 16777216 hep100 4194304
Prints GB/s, fraction of the measured copy, path and kernel per pair, worst first."""
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
KINDS = ["aos", "aos_aligned", "soa_sb", "soa_sb_aligned", "soa_mb", "aosoa4", "aosoa8", "aosoa32", "aosoa4_aligned",
         "split_p7", "split_pos", "split_hep"]
args = sys.argv[1:] or ["particle7", "16777216", "listing1", "16777216", "hep100", "4194304"]
rows = []
for schema, n in zip(args[::2], args[1::2]):
    n = int(n)
    sch = W.SCHEMAS[schema]
    maps = {}
    for k in KINDS:
        try:
            if k.startswith("split_") and not k.endswith({"particle7": "p7", "listing1": "pos", "hep100": "hep"}[schema]):
                continue
            maps[k] = llama.Mapping.from_spec(sch, [n], W.resolve_spec(k))
        except Exception:
            continue
    src = {k: m.alloc() for k, m in maps.items()}
    dst = {k: m.alloc() for k, m in maps.items()}
    for k, m in maps.items():
        llama.generate(m, src[k], 3)
    warm = time.time() + 0.3
    while time.time() < warm:
        llama.copy(maps["aos"], src["aos"], maps["soa_mb"], dst["soa_mb"])
        torch.cuda.synchronize()
    for a in maps:
        for b in maps:
            if a == b:
                continue
            sm, dm = maps[a], maps[b]
            llama.copy(sm, src[a], dm, dst[b])
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(10):
                llama.copy(sm, src[a], dm, dst[b])
            e1.record()
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1) / 10
            g = (sm.footprint() + dm.footprint()) / ms / 1e6
            pl = llama.plan(sm, dm)
            rows.append((g / PEAK, g, schema, n, a, b, pl["path"], pl["jit"]))
    del src, dst
    torch.cuda.empty_cache()
rows.sort()
for f, g, schema, n, a, b, path, jit in rows:
    print(f"{f:6.3f} {g:7.0f} GB/s  {schema:9s} {n:>9d}  {a:>15s} -> {b:<15s} {path}{' jit' if jit else ''}")
