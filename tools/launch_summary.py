#!/usr/bin/env python
"""Digests an ncu --csv launch list (gpu__time_duration / dram bytes per
launch) into per-kernel shares of the timed steps.  Usage:
    python tools/launch_summary.py launches.csv [--skip-prefix k_gen,k_fill]"""
import csv
import sys
from collections import OrderedDict


def main(path, skip=("k_gen", "k_fill")):
    rows = []
    with open(path) as f:
        lines = [l for l in f if l.startswith('"')]
    for r in csv.DictReader(lines):
        rows.append(r)
    launches = OrderedDict()
    for r in rows:
        key = r["ID"]
        d = launches.setdefault(key, {"name": r["Kernel Name"], "grid": r["Grid Size"]})
        d[r["Metric Name"]] = float(r["Metric Value"].replace(",", ""))
    ls = [v for v in launches.values() if not v["name"].startswith(skip)]
    tot = sum(v.get("gpu__time_duration.sum", 0) for v in ls)
    agg = OrderedDict()
    for v in ls:
        k = v["name"].split("(")[0]
        a = agg.setdefault(k, [0, 0.0, 0.0, 0.0])
        a[0] += 1
        a[1] += v.get("gpu__time_duration.sum", 0)
        a[2] += v.get("dram__bytes_read.sum", 0)
        a[3] += v.get("dram__bytes_write.sum", 0)
    print(f"{'kernel':32s} {'launches':>8s} {'avg_us':>9s} {'share':>7s} {'dram_rd_MB/launch':>18s} {'dram_wr_MB/launch':>18s}")
    for k, (n, t, rd, wr) in agg.items():
        unit = 1e-3 if t > 1e5 else 1.0  # ncu reports ns or us depending on version
        print(f"{k:32s} {n:8d} {t / n * unit:9.2f} {t / tot:7.1%} {rd / n / 1e6:18.1f} {wr / n / 1e6:18.1f}")
    print(f"total launches (excluding {','.join(skip)}): {len(ls)}")


if __name__ == "__main__":
    main(sys.argv[1])
