#!/usr/bin/env python
"""Staged-copy pipeline sweep: the bench's e2e step (16 C2 copies, pinned host
-> pinned host through llama_copy_staged_batch) at several slab sizes."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
if os.environ.get("LLAMA_PKG_ROOT"):
    sys.path.insert(0, os.environ["LLAMA_PKG_ROOT"])
import torch  # noqa: E402

import paper_2106_04284_b200 as llama  # noqa: E402
import workloads as W  # noqa: E402

cfg = W.CONFIGS["C2"]
schema = W.SCHEMAS[cfg["schema"]]
ext = list(cfg["extents"])
names = sorted({x for p in cfg["pairs"] for x in p})
maps = {k: llama.Mapping(schema, ext, *W.MAPPINGS[k]) for k in names}
hsrc = {k: [torch.empty(s, dtype=torch.uint8, pin_memory=True) for s in maps[k].blob_sizes()] for k in names}
hdst = {k: [torch.empty(s, dtype=torch.uint8, pin_memory=True) for s in maps[k].blob_sizes()] for k in names}
batch = [(maps[a], hsrc[a], maps[b], hdst[b]) for a, b in cfg["pairs"]]
nbytes = sum(maps[a].footprint() + maps[b].footprint() for a, b in cfg["pairs"])
for mib in [int(x) for x in (sys.argv[1] if len(sys.argv) > 1 else "32,64,128,256").split(",")]:
    st = llama.Stager(mib << 20)
    llama.copy_staged_batch(st, batch)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(2):
        llama.copy_staged_batch(st, batch)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 2
    print(f"slab {mib} MiB: {ms:.1f} ms {nbytes / ms / 1e6:.1f} GB/s", flush=True)
    del st
