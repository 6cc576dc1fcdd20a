#!/bin/bash
# A/B: old build (tools/ab_old) vs current on split + a few uniform pairs.
for rep in 1 2; do
 for v in ${VARIANTS:-old new}; do
  export LLAMA_WS_CONSUMERS=256; unset LLAMA_DST_BUFS LLAMA_WS_ORDER
  case $v in old) R=tools/ab_old;; exp) R=tools/ab_exp;; wide) R=; export LLAMA_WS_CONSUMERS=512;; nd3) R=; export LLAMA_DST_BUFS=3;; ord) R=; export LLAMA_WS_ORDER=1 LLAMA_DST_BUFS=2;; ord0) R=; export LLAMA_WS_ORDER=0 LLAMA_DST_BUFS=2;; ord2) R=; export LLAMA_WS_ORDER=2 LLAMA_DST_BUFS=2;; ord1nd3) R=; export LLAMA_WS_ORDER=1 LLAMA_DST_BUFS=3;; ord2nd3) R=; export LLAMA_WS_ORDER=2 LLAMA_DST_BUFS=3;; *) R=;; esac
  echo "== $v rep$rep"
  LLAMA_PKG_ROOT=$R python tools/split_ab.py aos:soa_mb,aos:aosoa8,aos:split_mb_a8,aos:split_mb_a32,split_mb_a8:aos,soa_mb:split_mb_a8 | awk '{print $1, $3, $(NF-3), $(NF-1)}'
  LLAMA_PKG_ROOT=$R python tools/profile_pairs.py --config C3 --records 8388608 --pairs aos:aos_aligned,aos:soa_mb,soa_mb:aos,aos_aligned:soa_mb,aos:split_hep --iters 3 | awk '{print $1, $3, $(NF-3), $(NF-1)}'
 done
done
for rep in 1; do
 for v in ${VARIANTS:-old new}; do
  export LLAMA_WS_CONSUMERS=256; unset LLAMA_DST_BUFS LLAMA_WS_ORDER
  case $v in old) R=tools/ab_old;; ord2) R=; export LLAMA_WS_ORDER=2 LLAMA_DST_BUFS=2;; *) R=;; esac
  echo "== $v rep$rep"
  LLAMA_PKG_ROOT=$R python tools/profile_pairs.py --config C4 --pairs aosoa32:soa_sb,aos:soa_sb,soa_sb:aos --iters 5 | awk '{print $1, $3, $(NF-3), $(NF-1)}'
  LLAMA_PKG_ROOT=$R python tools/profile_pairs.py --config C3 --records 8388608 --pairs aos:aos,soa_mb:soa_mb,aos_aligned:aos --iters 3 | awk '{print $1, $3, $(NF-3), $(NF-1)}'
 done
done
