#!/bin/bash
P=${PAIRS:-aos:soa_mb,aos:aosoa32,soa_mb:aos}
for dbg in 0 1 2 3; do
 for tb in 16384 24576 32768 49152; do
  for st in 2 4; do
      echo "== DEBUG=$dbg TILE_BYTES=$tb STAGES=$st"
      LLAMA_DEBUG_PERMUTE=$dbg LLAMA_TILE_BYTES=$tb LLAMA_STAGES=$st LLAMA_SMEM_BUDGET=230000 python tools/profile_pairs.py --pairs $P --iters 5
  done
 done
done
