#!/bin/bash
P=${PAIRS:-aos:soa_mb,aos:aosoa32,soa_mb:aos,aosoa8:aos}
for tb in 16384 24576 32768 49152 65536; do
  for st in 2 3; do
      echo "== TILE_BYTES=$tb STAGES=$st"
      LLAMA_TILE_BYTES=$tb LLAMA_STAGES=$st LLAMA_SMEM_BUDGET=230000 python tools/profile_pairs.py --pairs $P --iters 5
  done
done
