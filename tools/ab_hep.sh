#!/bin/bash
# HEP100 (C3 prefix) pairs under permute variants: old build vs current, warp-record mapping off/on, tile sizes.
P=aos:soa_mb,soa_mb:aos,aos_aligned:soa_mb,soa_mb:aos_aligned,aos:aos_aligned,aos_aligned:aos
run() { echo "== $1"; shift; env "$@" python tools/profile_pairs.py --config C3 --records 8388608 --pairs $P --iters 3 | awk '{print $1, $3, $(NF-3), $(NF-1)}'; }
run old LLAMA_PKG_ROOT=tools/ab_old
run new X=1
run nowmap LLAMA_WMAP=0
run t128 LLAMA_TILE_BYTES=98000 LLAMA_SMEM_BUDGET=230000
run t128s3 LLAMA_TILE_BYTES=98000 LLAMA_SMEM_BUDGET=230000 LLAMA_STAGES=2
