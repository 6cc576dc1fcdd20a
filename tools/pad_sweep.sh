set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_jit.py -x -q 2>&1 | tail -5 > gpurun_out/pad_tests.log
P1=aos:split_pos,split_pos:aos_aligned,soa_mb:split_pos,split_pos:aos,aos_aligned:split_pos,split_pos:soa_mb
for k in 0 1 2; do echo "== F1_listing1 jit_pad=$k"; timeout 300 python tools/profile_pairs.py --config C4 --records 67108864 --pairs $P1 --knobs jit_pad=$k --iters 5; done > gpurun_out/pad_sweep.txt 2>&1
P3=aos:aos_aligned,aos_aligned:aos,aos_aligned:soa_mb,soa_mb:aos_aligned
for k in 0 2; do echo "== C3 16M jit_pad=$k"; timeout 300 python tools/profile_pairs.py --config C3 --records 16777216 --pairs $P3 --knobs jit_pad=$k --iters 5; done >> gpurun_out/pad_sweep.txt 2>&1
cat gpurun_out/pad_tests.log gpurun_out/pad_sweep.txt
