# f4 block programs: JIT transpose parity (knobs), full-size f4 parity, then the knob sweep
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_jit.py -x -q -k "transpose" 2>&1 | tail -5 > gpurun_out/f4b_tests.log
timeout 900 python -m pytest tests/test_gpu_full_coverage.py -x -q -k "f4" 2>&1 | tail -3 >> gpurun_out/f4b_tests.log
timeout 900 python tools/f4_sweep.py > gpurun_out/f4b_sweep.txt 2>&1
cat gpurun_out/f4b_tests.log gpurun_out/f4b_sweep.txt
