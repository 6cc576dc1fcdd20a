#!/bin/bash
# One GPU call's worth of evidence for profiles/: bench lines (C2, MOVE), the
# ncu launch list of the C2 bench command, and --set full captures of the hot
# kernels (each command first run without ncu and checked for exit 0).
set -x
mkdir -p gpurun_out
python bench.py --steps 10 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err || exit 1
python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/b2.json 2>/dev/null || exit 1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv \
    --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/ncu_l.log 2>&1
python tools/profile_pairs.py --pairs aos:soa_mb,soa_mb:aos --iters 1 > /dev/null || exit 1
ncu --set full --clock-control none --import-source on -k regex:k_permute_ws -s 1 -c 1 -o gpurun_out/permute_full \
    python tools/profile_pairs.py --pairs aos:soa_mb --iters 1 > gpurun_out/ncu_p.log 2>&1
python tools/move_once.py > /dev/null || exit 1
ncu --set full --clock-control none --import-source on -k regex:k_move -c 3 -o gpurun_out/move_full \
    python tools/move_once.py > gpurun_out/ncu_m.log 2>&1
python bench.py --config MOVE --steps 10 --warmup 3 > gpurun_out/move.json 2> gpurun_out/move.err
ls -la gpurun_out
