#!/bin/bash
# Round-2 ncu evidence (each command first run without ncu):
#  1. DRAM bytes + duration of every launch of the dominant kernels of each
#     bench config (profiles/traffic.json is derived from it)
#  2. sector efficiency (global ld/st bytes per sector) of the LSU paths
set -x
mkdir -p gpurun_out
C2P=aos:aos,soa_mb:soa_mb,aosoa8:aosoa8,aosoa32:aosoa32,aos:soa_mb,soa_mb:aosoa8,aosoa8:aosoa32,aosoa32:aos,aos:aosoa8,soa_mb:aosoa32,aosoa8:aos,aosoa32:soa_mb,aos:aosoa32,soa_mb:aos,aosoa8:soa_mb,aosoa32:aosoa8
C3P=aos:aos_aligned,aos_aligned:soa_mb,soa_mb:aos,aos:soa_mb,soa_mb:aos_aligned,aos_aligned:aos
M="gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum"
python tools/profile_pairs.py --config C2 --iters 1 --pairs $C2P > /dev/null || exit 1
ncu --metrics $M --clock-control none --csv --log-file gpurun_out/r02_traffic_c2.csv python tools/profile_pairs.py --config C2 --iters 1 --pairs $C2P > /dev/null 2>&1
ncu --metrics $M --clock-control none --csv --log-file gpurun_out/r02_traffic_c4.csv python tools/profile_pairs.py --config C4 --iters 1 --pairs aosoa32:soa_sb > /dev/null 2>&1
ncu --metrics $M --clock-control none --csv --log-file gpurun_out/r02_traffic_c3.csv python tools/profile_pairs.py --config C3 --iters 1 --records 67108864 --pairs $C3P > /dev/null 2>&1
S="smsp__sass_average_data_bytes_per_sector_mem_global_op_ld.pct,smsp__sass_average_data_bytes_per_sector_mem_global_op_st.pct,l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum,dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum"
ncu --metrics $S --clock-control none --csv --log-file gpurun_out/r02_sectors.csv python tools/profile_pairs.py --config C2 --iters 1 --pairs aos:soa_mb,aosoa8:aosoa32 --path naive > /dev/null 2>&1
ncu --metrics $S --clock-control none --csv --log-file gpurun_out/r02_sectors_run.csv python tools/profile_pairs.py --config C2 --iters 1 --pairs aosoa8:aosoa32,soa_mb:aosoa32 --path run > /dev/null 2>&1
ncu --metrics $S --clock-control none --csv --log-file gpurun_out/r02_sectors_jit.csv python tools/profile_pairs.py --config C3 --records 16777216 --iters 1 --pairs aos:soa_mb,soa_mb:aos,aos:aos_aligned > /dev/null 2>&1
ncu --metrics $S --clock-control none --csv --log-file gpurun_out/r02_sectors_direct.csv python tools/profile_pairs.py --config C3 --records 16777216 --iters 1 --knobs jit=0 --pairs aos:soa_mb,soa_mb:aos > /dev/null 2>&1
ncu --metrics $S --clock-control none --csv --log-file gpurun_out/r02_sectors_ws.csv python tools/profile_pairs.py --config C2 --iters 1 --pairs aos:soa_mb,soa_mb:aos > /dev/null 2>&1
python tools/f4_bench.py > gpurun_out/f4_pre.txt 2>&1
ncu --metrics $S --clock-control none --csv --log-file gpurun_out/r02_sectors_f4.csv -k regex:k_transpose2d -c 6 python tools/f4_bench.py > /dev/null 2>&1
python tools/move_once.py > /dev/null || exit 1
ncu --metrics $M --clock-control none --csv --log-file gpurun_out/r02_traffic_move.csv -k regex:k_move_runs python tools/move_once.py > /dev/null 2>&1
ls -la gpurun_out/r02_*
