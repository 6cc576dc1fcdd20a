set -x
timeout 900 python -m pytest tests/test_gpu_jit.py tests/test_gpu_parity.py -x -q > gpurun_out/t3.log 2>&1; echo rc=$? >> gpurun_out/t3.log
P="--iters 5"
python tools/profile_pairs.py --config C4 --records 67108864 $P --pairs aos_aligned:split_pos,aos:split_pos,split_pos:aos,soa_mb:split_pos,aos_aligned:mapping_c > gpurun_out/split2.txt 2>&1
python tools/profile_pairs.py --config C4 --records 67108864 $P --knobs jit=2 --pairs aosoa32:soa_sb,aos:soa_mb,soa_mb:aos,aos:aos_aligned >> gpurun_out/split2.txt 2>&1
tail -3 gpurun_out/t3.log; cut -c1-30,190- gpurun_out/split2.txt
