#!/bin/bash
# Round-2 ncu traffic of every bench sub-config, pair by pair in bench.py's
# order (profiles/traffic.json via tools/traffic_from_ncu.py "csv:@CONFIG"),
# each command first run without ncu; plus sector efficiency of the JIT
# transposes (f4).
set -x
mkdir -p gpurun_out
M="gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum"
pairs() { python -c "import bench; print(','.join(a+':'+b for a,b in bench.pairs_of('$1')))"; }
run() {  # name, profile_pairs config, records
  local P; P=$(pairs $1)
  python tools/profile_pairs.py --config $2 --records $3 --iters 1 --pairs $P > gpurun_out/r02_pp_$1.txt 2>&1 || return 1
  ncu --metrics $M --clock-control none --csv --log-file gpurun_out/r02_traffic3_$1.csv \
    python tools/profile_pairs.py --config $2 --records $3 --iters 1 --pairs $P > /dev/null 2>&1
}
run C2 C2 16777216
run C2_soa_sb C2 16777216
run C3 C3 67108864
run C3_soa_sb C3 67108864
run F1_hep C3 16777216
run F1_listing1 C4 67108864
run C4_pairs C4 67108864
S="smsp__sass_average_data_bytes_per_sector_mem_global_op_ld.pct,smsp__sass_average_data_bytes_per_sector_mem_global_op_st.pct,l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum,dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum"
python tools/f4_sweep.py '[{}]' > gpurun_out/f4_pre3.txt 2>&1
ncu --metrics $S --clock-control none --csv --log-file gpurun_out/r02_sectors_f4_jit.csv -k regex:llb_jit python tools/f4_sweep.py '[{}]' > /dev/null 2>&1
ls -la gpurun_out/r02_traffic3_* gpurun_out/r02_sectors_f4_jit.csv
