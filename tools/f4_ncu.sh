# ncu --set full captures of the JIT transposes (after the same commands exit 0 without ncu)
mkdir -p gpurun_out
for c in "soa_mb col soa_mb row" "aos row aos col" "soa_mb morton aos col"; do python tools/f4_one.py $c >> gpurun_out/f4_one.txt 2>&1; done
i=0
for c in "soa_mb col soa_mb row" "aos row aos col" "soa_mb morton aos col"; do
  i=$((i+1))
  ncu --set full --clock-control none --import-source on -k regex:llb_jit -s 3 -c 1 -o gpurun_out/f4b_$i -f python tools/f4_one.py $c > gpurun_out/f4b_ncu_$i.log 2>&1
done
cat gpurun_out/f4_one.txt
