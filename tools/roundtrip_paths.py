#!/usr/bin/env python
"""Every copy path on small ragged inputs, self-checking without the oracle
(compute-sanitizer is not available on the GPU pool): each copy src -> dst is
followed by dst -> src' through the auto path and src' must equal src byte
for byte (round-trip identity; generated padding is 0 and destination padding
is written 0, DESIGN reading 12). Exit 1 on any mismatch."""
import itertools
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2106_04284_b200 as llama  # noqa: E402
import workloads as W  # noqa: E402

KINDS = ["aos", "aos_aligned", "soa_mb", "soa_sb", "aosoa4", "aosoa8", "aosoa32"]
CASES = [  # (schema, extents, linearizers)
    ("particle7", (4096 + 37,), ["row"]),
    ("listing1", (1000 + 13,), ["row"]),
    ("hep100", (640 + 21,), ["row"]),
    ("particle7", (67, 93), ["row", "col"]),
    ("particle7", (64, 64), ["row", "col", "morton"]),
]
PATHS = ["auto", "naive", "permute"]
bad = 0
runs = 0


def roundtrip(schema, ext, sspec, dspec, slin, dlin, path):
    global bad, runs
    sm = llama.Mapping.from_spec(W.SCHEMAS[schema], ext, W.resolve_spec(sspec), lin=slin)
    dm = llama.Mapping.from_spec(W.SCHEMAS[schema], ext, W.resolve_spec(dspec), lin=dlin)
    sb, db, rb = sm.alloc(), dm.alloc(), sm.alloc()
    llama.generate(sm, sb, 7)
    try:
        llama.copy(sm, sb, dm, db, path=None if path == "auto" else path)
    except llama.LlamaError as e:  # a forced path that does not apply to the pair
        if "UNSUPPORTED" in str(e) or "INVALID" in str(e):
            return
        raise
    llama.copy(dm, db, sm, rb)
    torch.cuda.synchronize()
    runs += 1
    if not all(torch.equal(a, b) for a, b in zip(sb, rb)):
        bad += 1
        print("MISMATCH", schema, ext, sspec, dspec, slin, dlin, path, llama.plan(sm, dm))


for schema, ext, lins in CASES:
    for s, d in itertools.product(KINDS, KINDS):
        for slin, dlin in itertools.product(lins, lins):
            if len(lins) > 1 and s != d and (slin, dlin) != ("row", "row"):
                continue  # transposes: equal kinds only, to keep the run short
            for path in PATHS:
                roundtrip(schema, ext, s, d, slin, dlin, path)
for name, (schema, spec) in W.SPLITS.items():
    if "one" in repr(spec):
        continue  # a One part maps many records onto one location: no copy into it, no round trip
    ext = (1000 + 29,) if schema != "hep100" else (300 + 7,)
    for other in ["aos", "soa_mb", "aosoa8"]:
        roundtrip(schema, ext, name, other, "row", "row", "auto")
        roundtrip(schema, ext, other, name, "row", "row", "auto")

# staged host <-> device relayout (f2)
sm = llama.Mapping.from_spec(W.PARTICLE7, (100_003,), W.resolve_spec("aos"))
dm = llama.Mapping.from_spec(W.PARTICLE7, (100_003,), W.resolve_spec("soa_mb"))
sb, db = sm.alloc(), dm.alloc()
llama.generate(sm, sb, 3)
llama.copy(sm, sb, dm, db)
hs = [b.cpu().pin_memory() for b in sb]
hd = [torch.empty(b.numel(), dtype=torch.uint8).pin_memory() for b in db]
st = llama.Stager(slab_bytes=1 << 20)
llama.copy_staged(st, sm, hs, dm, hd)
torch.cuda.synchronize()
runs += 1
if not all(torch.equal(a.cpu(), b) for a, b in zip(db, hd)):
    bad += 1
    print("MISMATCH staged")

# n-body move (f3): every move path on each layout, then compare layouts via copy
ref = None
for spec in ["aos", "soa_mb", "aosoa8"]:
    for mp in ["auto", "generic"]:
        m = llama.Mapping.from_spec(W.PARTICLE7, (4096 + 5,), W.resolve_spec(spec))
        b = m.alloc()
        llama.generate(m, b, 11)
        llama.nbody_move(m, b, W.NBODY_TIMESTEP, path=mp)
        am = llama.Mapping.from_spec(W.PARTICLE7, (4096 + 5,), W.resolve_spec("aos"))
        ab = am.alloc()
        llama.copy(m, b, am, ab)
        torch.cuda.synchronize()
        runs += 1
        if ref is None:
            ref = ab[0].clone()
        elif not torch.equal(ref, ab[0]):
            bad += 1
            print("MISMATCH move", spec, mp)

print(f"roundtrip_paths: {runs} checks, {bad} mismatches, {llama.launch_count()} launches")
sys.exit(1 if bad else 0)
