#!/bin/bash
# A/B over the 16 C2 pairs: old build (tools/ab_old) vs current, alternating, same box.
P=aos:aos,aos:soa_mb,aos:aosoa8,aos:aosoa32,soa_mb:aos,soa_mb:soa_mb,soa_mb:aosoa8,soa_mb:aosoa32,aosoa8:aos,aosoa8:soa_mb,aosoa8:aosoa8,aosoa8:aosoa32,aosoa32:aos,aosoa32:soa_mb,aosoa32:aosoa8,aosoa32:aosoa32
for rep in 1 2; do  # VARIANTS='old exp new' adds tools/ab_exp
 for v in ${VARIANTS:-old new}; do
  export LLAMA_WS_CONSUMERS=256; unset LLAMA_DST_BUFS LLAMA_WS_ORDER
  case $v in old) R=tools/ab_old;; exp) R=tools/ab_exp;; wide) R=; export LLAMA_WS_CONSUMERS=512;; nd3) R=; export LLAMA_DST_BUFS=3;; ord) R=; export LLAMA_WS_ORDER=1 LLAMA_DST_BUFS=2;; ord0) R=; export LLAMA_WS_ORDER=0 LLAMA_DST_BUFS=2;; ord2) R=; export LLAMA_WS_ORDER=2 LLAMA_DST_BUFS=2;; ord1nd3) R=; export LLAMA_WS_ORDER=1 LLAMA_DST_BUFS=3;; ord2nd3) R=; export LLAMA_WS_ORDER=2 LLAMA_DST_BUFS=3;; *) R=;; esac
  echo "== $v rep$rep"
  LLAMA_PKG_ROOT=$R python tools/profile_pairs.py --pairs $P --iters 10 | awk '{print $1, $3, $(NF-3), $(NF-1)}'
 done
done
