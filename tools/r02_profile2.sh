#!/bin/bash
# Round-2 full ncu captures of the final JIT kernels (each command first run without ncu):
# llb_jit_permute on HEP100 SoA MB -> packed AoS and packed AoS -> SoA MB (16M records),
# llb_jit_transpose on Particle7 AoS col -> row (4096^2)
set -x
mkdir -p gpurun_out
python tools/profile_pairs.py --config C3 --records 16777216 --iters 1 --pairs soa_mb:aos,aos:soa_mb > /dev/null || exit 1
ncu --set full --clock-control none --import-source on -k regex:llb_jit -s 1 -c 1 -o gpurun_out/r02_jit_s2a python tools/profile_pairs.py --config C3 --records 16777216 --iters 1 --pairs soa_mb:aos > gpurun_out/ncu_j1.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:llb_jit -s 1 -c 1 -o gpurun_out/r02_jit_a2s python tools/profile_pairs.py --config C3 --records 16777216 --iters 1 --pairs aos:soa_mb > gpurun_out/ncu_j2.log 2>&1
python tools/transpose_once.py aos > /dev/null || exit 1
ncu --set full --clock-control none --import-source on -k regex:llb_jit -s 1 -c 1 -o gpurun_out/r02_t2d python tools/transpose_once.py aos > gpurun_out/ncu_j3.log 2>&1
ls -la gpurun_out/r02_*.ncu-rep
