import sys, torch
sys.path.insert(0, '.')
import paper_2106_04284_b200 as llama, workloads as W
n = 1 << 24
sm = llama.Mapping.from_spec(W.LISTING1, [n], W.resolve_spec("aos"))
dm = llama.Mapping.from_spec(W.LISTING1, [n], W.resolve_spec("soa_mb"))
big = torch.empty(3 << 30, dtype=torch.uint8, device="cuda")
def views(m, off):
    out, o = [], off
    for x in m.blob_sizes():
        out.append(big[o:o + x]); o += (x + 4095) // 4096 * 4096
    return out, o
sb, end = views(sm, 0)
llama.generate(sm, sb, 1)
for doff in [end, end + 4096, end + 65536, end + (1 << 20), end + (1 << 21), end + (1 << 22) + 8192, end + (3 << 20), end + (1 << 24)]:
    doff = (doff + 255) // 256 * 256
    db, _ = views(dm, doff)
    for _ in range(20): llama.copy(sm, sb, dm, db)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    res = []
    for pair in ((sm, sb, dm, db), (dm, db, sm, sb)):
        e0.record()
        for _ in range(20): llama.copy(*pair)
        e1.record(); torch.cuda.synchronize()
        res.append((sm.footprint() + dm.footprint()) / (e0.elapsed_time(e1) / 20) / 1e6)
    print(f"dst offset {doff - end:>10d}: aos->soa_mb {res[0]:.0f}  soa_mb->aos {res[1]:.0f} GB/s", flush=True)
