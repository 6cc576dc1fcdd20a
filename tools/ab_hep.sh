#!/bin/bash
# HEP100 (C3 prefix) pairs: variants.
P=soa_mb:aos,soa_mb:aos_aligned,aos:soa_mb,aos_aligned:soa_mb
run() { echo "== $1"; shift; env "$@" python tools/profile_pairs.py --config C3 --records 8388608 --pairs $P --iters 3 | awk '{print $1, $3, $(NF-3), $(NF-1)}'; }
run permute LLAMA_DIRECT_REPACK=0
run repack X=1
run permute2 LLAMA_DIRECT_REPACK=0
run repack2 X=1
