#!/bin/bash
# Direct permute consumer-count variants (tools/ab_exp/c<cons>_<minblocks>, git-ignored builds)
# against the working tree on HEP100 (C3 prefix), alternating on one box.
P=${PAIRS:-soa_mb:aos,soa_mb:aos_aligned,aos:soa_mb,aos_aligned:soa_mb}
for rep in 1 2; do
  for R in "" tools/ab_exp/c384_2 tools/ab_exp/c512_2 tools/ab_exp/c384_3; do
    echo "== ${R:-base} rep$rep"
    LLAMA_PKG_ROOT=$R python tools/profile_pairs.py --config C3 --records 8388608 --pairs $P --iters 3 | awk '{print $1, $3, $(NF-3), $(NF-1)}'
  done
done
