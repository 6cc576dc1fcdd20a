#!/bin/bash
# HEP100 (C3 prefix) pairs under permute variants.
P=aos:soa_mb,aos:soa_sb,aos_aligned:soa_mb,soa_mb:aos
run() { echo "== $1"; shift; env "$@" python tools/profile_pairs.py --config C3 --records 8388608 --pairs $P --iters 3 | awk '{print $1, $3, $(NF-3), $(NF-1)}'; }
run new X=1
run forced LLAMA_DIRECT=2
