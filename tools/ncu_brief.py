#!/usr/bin/env python
"""Short summary of an ncu --set full report (one kernel): duration, DRAM and
issue utilisation, occupancy, the top stall reasons, shared-memory wavefronts
and bank conflicts, L2 / DRAM bytes.  python tools/ncu_brief.py rep.ncu-rep ..."""
import csv
import io
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "dram__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__inst_executed.avg.per_cycle_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "launch__occupancy_limit_shared_mem", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
        "smsp__inst_executed.sum", "lts__t_bytes.sum"]


def main(paths):
    for p in paths:
        out = subprocess.run(["ncu", "-i", p, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
        rows = list(csv.reader(io.StringIO(out)))
        h, units, v = rows[0], rows[1], rows[2]
        d = dict(zip(h, v))
        u = dict(zip(h, units))
        print("==", p, d.get("Kernel Name", "")[:60])
        for k in KEYS:
            if k in d:
                print(f"  {k} = {d[k]} {u.get(k, '')}")
        st = []
        for k in d:
            if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued"):
                try:
                    st.append((float(d[k].replace(",", "")), k[len("smsp__pcsamp_warps_issue_stalled_"):]))
                except ValueError:
                    pass
        tot = sum(x for x, _ in st) or 1
        print("  stalls: " + ", ".join(f"{n} {x / tot:.0%}" for x, n in sorted(st, reverse=True)[:7]))


if __name__ == "__main__":
    main(sys.argv[1:])
