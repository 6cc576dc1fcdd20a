#!/bin/bash
# HEP100 AoS <-> aligned AoS (tile permute, word mode): tile / budget / stages / dst-buffer sweep.
P=aos:aos_aligned,aos_aligned:aos
run() { echo "== $*"; env "$@" python tools/profile_pairs.py --config C3 --records 8388608 --pairs $P --iters 3 | awk '{print $1, $3, $4, $(NF-1)}'; }
run X=1
for tb in 24576 32768 49152 65536 98304; do run LLAMA_TILE_BYTES=$tb; done
for sb in 80000 150000 230000; do run LLAMA_SMEM_BUDGET=$sb; done
for st in 2 3 4; do run LLAMA_STAGES=$st; done
for db in 2 3 4; do run LLAMA_DST_BUFS=$db; done
for o in 0 1; do run LLAMA_WS_ORDER=$o; done
run X=1
