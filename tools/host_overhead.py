#!/usr/bin/env python
"""Host cost of one llama.copy call through the Python binding (tiny copies,
so the GPU never limits): microseconds per call by argument style."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2106_04284_b200 as llama  # noqa: E402
import workloads as W  # noqa: E402

for schema, a, b in (("particle7", "aos", "soa_mb"), ("listing1", "soa_mb", "aos"), ("hep100", "aos", "soa_mb")):
    sm = llama.Mapping.from_spec(W.SCHEMAS[schema], [256], W.resolve_spec(a))
    dm = llama.Mapping.from_spec(W.SCHEMAS[schema], [256], W.resolve_spec(b))
    sb, db = sm.alloc(), dm.alloc()
    for label, kw in (("plain", {}), ("path", {"path": "permute"}), ("knobs", {"knobs": {"stages": 3}})):
        for _ in range(50):
            llama.copy(sm, sb, dm, db, **kw)
        torch.cuda.synchronize()
        t = time.perf_counter()
        for _ in range(2000):
            llama.copy(sm, sb, dm, db, **kw)
        dt = (time.perf_counter() - t) / 2000 * 1e6
        torch.cuda.synchronize()
        print(f"{schema:9s} {a}->{b} {label:6s} {dt:7.1f} us/call (host, {sm.blob_count}+{dm.blob_count} blobs)")
