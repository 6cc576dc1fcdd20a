#!/bin/bash
# HEP100 (C3 prefix) pairs under permute variants.
P=aos:soa_mb,soa_mb:aos,aos_aligned:soa_mb,soa_mb:aos_aligned,aos:aos_aligned,aos_aligned:aos
run() { echo "== $1"; shift; env "$@" python tools/profile_pairs.py --config C3 --records 8388608 --pairs $P --iters 3 | awk '{print $1, $3, $(NF-3), $(NF-1)}'; }
run old LLAMA_PKG_ROOT=tools/ab_old
run ns2 X=1
run ns3 LLAMA_DIRECT_STAGES=3
run ns4 LLAMA_DIRECT_STAGES=4
