#!/bin/bash
# HEP100 AoS <-> SoA MB (direct permute): knob sweep on the final code.
P=soa_mb:aos,soa_mb:aos_aligned,aos:soa_mb,aos_aligned:soa_mb
run() { echo "== $*"; env "$@" python tools/profile_pairs.py --config C3 --records 8388608 --pairs $P --iters 3 | awk '{print $1, $3, $(NF-1)}'; }
run X=1
for st in 3 4; do run LLAMA_DIRECT_STAGES=$st; done
run LLAMA_DIRECT_ASYNC=0
run LLAMA_DIRECT_PHASE=0
run LLAMA_DIRECT_STAGING=0
run LLAMA_DIRECT_CHUNKS=0
run LLAMA_DIRECT=0
run X=1
