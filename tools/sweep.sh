#!/bin/bash
# Tile/stage/TMA sweep of the permute path on C2 pairs (one GPU).
P=${PAIRS:-aos:soa_mb,aos:aosoa32,soa_mb:aos}
for tb in 12288 24576 49152 98304; do
  for st in 2 3 4; do
    for bud in 80000 112000 220000; do
      echo "== TILE_BYTES=$tb STAGES=$st BUDGET=$bud"
      LLAMA_TILE_BYTES=$tb LLAMA_STAGES=$st LLAMA_SMEM_BUDGET=$bud python tools/profile_pairs.py --pairs $P --iters 5
    done
  done
done
echo "== NO_TMA"
LLAMA_NO_TMA=1 python tools/profile_pairs.py --pairs $P --iters 5
