#!/usr/bin/env python
"""Summarises an ncu report: per launch the key throughput / traffic metrics
and the top warp stall reasons.  Usage: python tools/ncu_summary.py rep.ncu-rep"""
import csv
import io
import subprocess
import sys

KEYS = ["Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "l1tex__throughput.avg.pct_of_peak_sustained_active", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "launch__grid_size", "launch__occupancy_limit_shared_mem",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smsp__inst_executed.sum",
        "smsp__sass_average_data_bytes_per_sector_mem_global_op_ld.pct",
        "smsp__sass_average_data_bytes_per_sector_mem_global_op_st.pct"]


def main(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    for r in rows[2:]:
        print("=" * 100)
        for k in KEYS:
            if k in hdr:
                i = hdr.index(k)
                print(f"  {k:70s} {r[i]} {units[i]}")
        stalls = []
        pre = "smsp__average_warps_issue_stalled_"
        for i, h in enumerate(hdr):
            if h.startswith(pre) and h.endswith("_per_issue_active.ratio"):
                try:
                    stalls.append((float(r[i]), h[len(pre):-len("_per_issue_active.ratio")]))
                except ValueError:
                    pass
        stalls.sort(reverse=True)
        print("  top stalls (warps stalled per issue):", ", ".join(f"{n}={v:.2f}" for v, n in stalls[:8]))


if __name__ == "__main__":
    for p in sys.argv[1:]:
        main(p)
