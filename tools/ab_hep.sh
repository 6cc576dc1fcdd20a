#!/bin/bash
# HEP100 (C3 prefix) pairs: environment-knob variants of the working tree, alternating.
P=${PAIRS:-soa_mb:aos,soa_mb:aos_aligned,aos:soa_mb,aos_aligned:soa_mb}
run() { echo "== $1"; shift; env "$@" python tools/profile_pairs.py --config C3 --records 8388608 --pairs $P --iters 3 | awk '{print $1, $3, $(NF-3), $(NF-1)}'; }
for rep in 1 2; do
  run "${A_NAME:-a}" ${A_ENV:-X=1}
  run "${B_NAME:-b}" ${B_ENV:-X=1}
done
