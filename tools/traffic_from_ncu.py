#!/usr/bin/env python
"""Builds profiles/traffic.json (DRAM bytes per launch of each bench config's
dominant kernel, keyed "config/kernel") from the ncu launch lists that
tools/r02_profile.sh writes:
    python tools/traffic_from_ncu.py gpurun_out/r02_traffic_c2.csv:C2 gpurun_out/r02_traffic_c3.csv:C3 ...
Per kernel: mean dram read + write bytes per launch, mean duration, and the
cold-cache fraction = algorithmic bytes per launch / duration / measured peak
(the bench's algorithmic bytes: source + destination footprint)."""
import csv
import json
import os
import sys
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
ALGO = {"C2": 939524096, "C2_soa_sb": 939524096, "C4": 2818572288,
        "MOVE": 36 * (1 << 28)}  # n-body move: 24 B read + 12 B written per particle, 256Mi particles
C3_BYTES = {"aos:aos_aligned": 57713623040, "aos_aligned:soa_mb": 57713623040, "soa_mb:aos": 51002736640,
            "aos:soa_mb": 51002736640, "soa_mb:aos_aligned": 57713623040, "aos_aligned:aos": 57713623040}


def short(name):
    for k in ("llb_jit_permute", "llb_jit_transpose", "k_transpose_wide", "k_permute_ws", "k_permute_direct",
              "k_bulkcopy", "k_run", "k_naive", "k_transpose2d", "k_gen", "k_fill", "k_move_runs", "k_move_aos_tma"):
        if k in name:
            return k
    return name.split("(")[0]


def load(path):
    rows = [r for r in csv.reader(open(path)) if r]
    start = next(i for i, r in enumerate(rows) if "Metric Name" in r)
    hdr = rows[start]
    idx = {h: i for i, h in enumerate(hdr)}
    launches = defaultdict(dict)
    for r in rows[start + 1:]:
        if len(r) < len(hdr):
            continue
        key = (r[idx["ID"]], r[idx["Kernel Name"]])
        v = r[idx["Metric Value"]].replace(",", "")
        unit = r[idx["Metric Unit"]]
        try:
            x = float(v)
        except ValueError:
            continue
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-9, "usecond": 1e-6, "ns": 1e-9,
                 "us": 1e-6, "ms": 1e-3, "s": 1.0,
                 "msecond": 1e-3, "second": 1.0}.get(unit, 1.0)
        launches[key][r[idx["Metric Name"]]] = x * scale
    return launches


def pair_bytes(cfg):
    """Algorithmic bytes (source + destination footprint) of each pair of a
    bench sub-config, in bench.py's pair order (bench.SUBCFG / pairs_of)."""
    sys.path.insert(0, ROOT)
    import bench
    import paper_2106_04284_b200 as llama
    import workloads as W
    sc = bench.SUBCFG[cfg]
    schema = W.SCHEMAS[sc["schema"]]
    out = []
    def view(spec):  # kind or kind/linearisation (F4 sub-configs)
        kind, _, lin = spec.partition("/")
        return llama.Mapping.from_spec(schema, sc["extents"], W.resolve_spec(kind), lin=lin or "row")
    for a, b in bench.pairs_of(cfg):
        out.append(view(a).footprint() + view(b).footprint())
    return out


def main(args):
    peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]
    out = {}
    for spec in args:
        path, cfg = spec.split(":")
        launches = load(path)
        if cfg.startswith("@"):  # a bench sub-config run pair by pair (tools/r02_profile3.sh): per-launch bytes
            cfg = cfg[1:]
            pb = pair_bytes(cfg)
            copies = [(name, m) for (lid, name), m in sorted(launches.items(), key=lambda kv: int(kv[0][0]))
                      if short(name) not in ("k_gen", "k_fill")]
            timed = copies[1::2]  # warm-up + timed launch per pair
            per = defaultdict(list)
            for j, (name, m) in enumerate(timed[:len(pb)]):
                per[short(name)].append((m, pb[j]))
            for k, ms in per.items():
                dram = sum(m.get("dram__bytes_read.sum", 0) + m.get("dram__bytes_write.sum", 0) for m, _ in ms) / len(ms)
                dur = sum(m.get("gpu__time_duration.sum", 0) for m, _ in ms) / len(ms)
                algo = sum(b for _, b in ms) / len(ms)
                out[f"{cfg}/{k}"] = {
                    "launches": len(ms), "dram_bytes_per_launch": dram,
                    "dram_read_per_launch": sum(m.get("dram__bytes_read.sum", 0) for m, _ in ms) / len(ms),
                    "dram_write_per_launch": sum(m.get("dram__bytes_write.sum", 0) for m, _ in ms) / len(ms),
                    "duration_s_per_launch": dur, "algorithmic_bytes_per_launch": algo,
                    "cold_frac": algo / dur / 1e9 / peak, "dram_over_algorithmic": dram / algo,
                    "source": f"{os.path.basename(path)} (ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,"
                              "gpu__time_duration.sum --clock-control none; tools/r02_profile3.sh)"}
            continue
        per = defaultdict(list)
        for (lid, name), m in sorted(launches.items(), key=lambda kv: int(kv[0][0])):
            per[short(name)].append(m)
        for k, ms in per.items():
            if k in ("k_gen", "k_fill"):
                continue
            # profile_pairs runs every pair twice (warm-up + timed): keep the timed launches
            if cfg != "MOVE":
                ms = ms[1::2] if len(ms) % 2 == 0 and len(ms) > 1 else ms
            dram = [m.get("dram__bytes_read.sum", 0) + m.get("dram__bytes_write.sum", 0) for m in ms]
            dur = [m.get("gpu__time_duration.sum", 0) for m in ms]
            algo = ALGO.get(cfg) if cfg != "C3" else sum(C3_BYTES.values()) / len(C3_BYTES)
            e = {"launches": len(ms), "dram_bytes_per_launch": sum(dram) / len(dram),
                 "dram_read_per_launch": sum(m.get("dram__bytes_read.sum", 0) for m in ms) / len(ms),
                 "dram_write_per_launch": sum(m.get("dram__bytes_write.sum", 0) for m in ms) / len(ms),
                 "duration_s_per_launch": sum(dur) / len(dur), "source": f"{os.path.basename(path)} (ncu --metrics "
                 "dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none; "
                 "tools/r02_profile.sh)"}
            if algo:
                e["algorithmic_bytes_per_launch"] = algo
                e["cold_frac"] = algo / e["duration_s_per_launch"] / 1e9 / peak
                e["dram_over_algorithmic"] = e["dram_bytes_per_launch"] / algo
            out[f"{cfg}/{k}"] = e
    dst = os.path.join(ROOT, "profiles", "traffic.json")
    old = json.load(open(dst)) if os.path.exists(dst) else {}
    old = {k: v for k, v in old.items() if "/" in k}  # drop round-1 keys (not keyed by config)
    old.update(out)
    json.dump(old, open(dst, "w"), indent=1, sort_keys=True)
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main(sys.argv[1:])
