# sector efficiency and shared-memory wavefronts of the wide kernel's LSU accesses, one pair per mode
mkdir -p gpurun_out
S="smsp__sass_average_data_bytes_per_sector_mem_global_op_ld.pct,smsp__sass_average_data_bytes_per_sector_mem_global_op_st.pct,l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum,dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum"
CASES=("hep100 1024 soa_mb/row soa_mb/col" "hep100 1024 soa_mb/col aos/row" "hep100 1024 aos/row soa_mb/col" "hep100 1024 aos/row aos/morton" "hep100 1024 aosoa8/row aosoa8/col")
for c in "${CASES[@]}"; do python tools/wide_once.py $c > /dev/null 2>&1 || exit 1; done
for c in "${CASES[@]}"; do
  echo "== $c"
  ncu --metrics $S --clock-control none --csv -k regex:k_transpose_wide -s 3 -c 1 python tools/wide_once.py $c 2>/dev/null | grep -E '"(smsp|l1tex|dram|gpu__)' | awk -F'","' '{print $(NF-2), $NF}' | tr -d '"'
done
