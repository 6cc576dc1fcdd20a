#!/bin/bash
for rep in 1 2; do
 for v in old v1 ws; do
  R=; V1=0
  if [ $v = old ]; then R=tools/ab_old; fi
  if [ $v = v1 ]; then V1=1; fi
  echo "== $v rep$rep"
  LLAMA_PERMUTE_V1=$V1 LLAMA_PKG_ROOT=$R python tools/profile_pairs.py --pairs aos:soa_mb,soa_mb:aos,aos:aosoa8,aosoa8:aosoa32,aosoa32:aos --iters 10
  LLAMA_PERMUTE_V1=$V1 LLAMA_PKG_ROOT=$R python tools/profile_pairs.py --config C3 --records 16777216 --pairs aos:aos_aligned,aos:soa_mb,aos_aligned:soa_mb --iters 3
  LLAMA_PERMUTE_V1=$V1 LLAMA_PKG_ROOT=$R python tools/profile_pairs.py --config C4 --pairs aosoa32:soa_sb --iters 5
 done
done
