#!/bin/bash
# HEP100 (C3 prefix) pairs under permute variants.
P=aos_aligned:soa_mb,soa_mb:aos_aligned,aos:soa_mb,soa_mb:aos,aos:soa_sb
run() { echo "== $1"; shift; env "$@" python tools/profile_pairs.py --config C3 --records 8388608 --pairs $P --iters 3 | awk '{print $1, $3, $(NF-3), $(NF-1)}'; }
run nomix LLAMA_DIRECT_MIX=0
run mix X=1
run nomix2 LLAMA_DIRECT_MIX=0
run mix2 X=1
