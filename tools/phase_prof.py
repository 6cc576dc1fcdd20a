#!/usr/bin/env python
"""Phase timers of k_permute (LLAMA_DEBUG_PERMUTE=4): average cycles per tile
spent by thread 0 in each phase.  Usage: LLAMA_DEBUG_PERMUTE=4 python tools/phase_prof.py --config C3 --pairs aos:soa_mb"""
import argparse, ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2106_04284_b200 as llama
import workloads as W
ap = argparse.ArgumentParser()
ap.add_argument("--config", default="C2"); ap.add_argument("--pairs", default="aos:soa_mb")
ap.add_argument("--records", type=int, default=0)
a = ap.parse_args()
cfg = W.CONFIGS[a.config]; schema = W.SCHEMAS[cfg["schema"]]
ext = [a.records] if a.records else list(cfg["extents"])
f = llama.lib().llama_debug_permute_profile
f.argtypes = [ctypes.POINTER(ctypes.c_ulonglong), ctypes.c_int]
for pair in a.pairs.split(","):
    s, d = pair.split(":")
    sm, dm = llama.Mapping(schema, ext, *W.MAPPINGS[s]), llama.Mapping(schema, ext, *W.MAPPINGS[d])
    sb, db = sm.alloc(), dm.alloc()
    llama.generate(sm, sb, 42)
    llama.copy(sm, sb, dm, db); torch.cuda.synchronize()
    buf = (ctypes.c_ulonglong * 8)(); f(buf, 1)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); llama.copy(sm, sb, dm, db); e1.record(); torch.cuda.synchronize()
    f(buf, 1)
    n = max(1, buf[5])
    ms = e0.elapsed_time(e1)
    print(f"{s}->{d} {llama.plan(sm, dm)} {ms:.3f} ms {(sm.footprint()+dm.footprint())/ms/1e6:.0f} GB/s tiles(cta0 measured)={n}")
    names = ["mbar_wait", "drain+barA", "permute+fence(t0)", "barB", "issue"]
    print("   cycles/tile:", ", ".join(f"{nm}={buf[j]/n:.0f}" for j, nm in enumerate(names)), f"fence={buf[6]/n:.0f}")
    del sb, db
