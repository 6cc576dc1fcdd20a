# ncu --set full captures of the wide transposing copy, one per mode (after the same commands exit 0 without ncu)
mkdir -p gpurun_out
CASES=("hep100 1024 soa_mb/row soa_mb/col" "hep100 1024 soa_mb/col aos/row" "hep100 1024 aos/row soa_mb/col" "hep100 1024 aos/row aos_aligned/col" "hep100 1024 aos/row aos/morton")
for c in "${CASES[@]}"; do python tools/wide_once.py $c >> gpurun_out/wide_once.txt 2>&1 || exit 1; done
i=0
for c in "${CASES[@]}"; do
  i=$((i+1))
  ncu --set full --clock-control none --import-source on -k regex:k_transpose_wide -s 3 -c 1 -o gpurun_out/wide_$i -f python tools/wide_once.py $c > gpurun_out/wide_ncu_$i.log 2>&1
done
cat gpurun_out/wide_once.txt
