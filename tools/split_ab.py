#!/usr/bin/env python
"""Times the tile permute for Particle7 split layouts against uniform ones
(where the split's cost comes from: parts vs intra-part layout)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
if os.environ.get("LLAMA_PKG_ROOT"):  # A/B against another build of the package
    sys.path.insert(0, os.environ["LLAMA_PKG_ROOT"])
import torch  # noqa: E402

import paper_2106_04284_b200 as llama  # noqa: E402
import workloads as W  # noqa: E402

N = 1 << 24
S = W.PARTICLE7
SPECS = {
    "aos": ("aos", 1, False), "soa_mb": ("soa_mb", 1, False), "aosoa8": ("aosoa", 8, False), "aosoa32": ("aosoa", 32, False),
    "split_mb_mb": ([0, 1, 2], ("soa_mb", 1, False), ("soa_mb", 1, False)),
    "split_mb_aos": ([0, 1, 2], ("soa_mb", 1, False), ("aos", 1, False)),
    "split_mb_a8": ([0, 1, 2], ("soa_mb", 1, False), ("aosoa", 8, False)),
    "split_mb_a32": ([0, 1, 2], ("soa_mb", 1, False), ("aosoa", 32, False)),
    "split_aos_aos": ([0, 1, 2], ("aos", 1, False), ("aos", 1, False)),
}
pairs = sys.argv[1].split(",") if len(sys.argv) > 1 else [
    "aos:soa_mb", "aos:aosoa8", "aos:split_mb_mb", "aos:split_mb_aos", "aos:split_mb_a8", "aos:split_mb_a32",
    "aos:split_aos_aos", "split_mb_a8:aos", "soa_mb:split_mb_a8"]
for pr in pairs:
    a, b = pr.split(":")
    sm = llama.Mapping.from_spec(S, [N], SPECS[a])
    dm = llama.Mapping.from_spec(S, [N], SPECS[b])
    sb, db = sm.alloc(), dm.alloc()
    llama.generate(sm, sb, 1)
    llama.copy(sm, sb, dm, db)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        llama.copy(sm, sb, dm, db)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 5
    info = llama.plan(sm, dm)
    print(f"{a:>14} -> {b:<14} {info['path']:8s} T={info['tile_records']:5d} smem={info['smem_bytes']:6d} "
          f"{ms:.3f} ms {(sm.footprint() + dm.footprint()) / ms / 1e6:.0f} GB/s", flush=True)
