#!/bin/bash
# HEP100 (C3 prefix) pairs: old build vs current.
P=soa_mb:aos_aligned,aos:soa_mb,aos_aligned:soa_mb,aos:soa_sb
run() { echo "== $1"; shift; env "$@" python tools/profile_pairs.py --config C3 --records 8388608 --pairs $P --iters 3 | awk '{print $1, $3, $(NF-3), $(NF-1)}'; }
run old LLAMA_PKG_ROOT=tools/ab_old
run new X=1
run old2 LLAMA_PKG_ROOT=tools/ab_old
run new2 X=1
