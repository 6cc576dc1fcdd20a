#!/bin/bash
# HEP100 (C3 prefix) pairs under permute variants.
P=soa_mb:aos_aligned,aos:soa_mb,aos_aligned:soa_mb,aos:soa_sb
run() { echo "== $1"; shift; env "$@" python tools/profile_pairs.py --config C3 --records 8388608 --pairs $P --iters 3 | awk '{print $1, $3, $(NF-3), $(NF-1)}'; }
run new X=1
run ns2 LLAMA_DIRECT_STAGES=2
run new2 X=1
