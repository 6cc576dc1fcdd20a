#!/bin/bash
# A/B: old build (tools/ab_old) vs current, alternating, same box.
for rep in 1 2; do
 for v in old new; do
  if [ $v = old ]; then R=tools/ab_old; else R=; fi
  echo "== $v rep$rep"
  LLAMA_PKG_ROOT=$R python tools/profile_pairs.py --pairs aos:soa_mb,soa_mb:aos,aos:aosoa8,aosoa8:aosoa32 --iters 10
  LLAMA_PKG_ROOT=$R python tools/profile_pairs.py --config C3 --records 16777216 --pairs aos:aos_aligned,aos:soa_mb --iters 3
  LLAMA_PKG_ROOT=$R python tools/profile_pairs.py --config C4 --pairs aosoa32:soa_sb --iters 5
 done
done
