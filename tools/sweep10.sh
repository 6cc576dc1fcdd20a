#!/bin/bash
PAIRS=aos:aos_aligned,aos:soa_mb,aos_aligned:soa_mb
for st in 2 3 4; do for bud in 75000 120000 230000; do for tb in 24576 49152; do
  echo "== C3 ST=$st BUD=$bud TB=$tb"
  LLAMA_STAGES=$st LLAMA_SMEM_BUDGET=$bud LLAMA_TILE_BYTES=$tb python tools/profile_pairs.py --config C3 --pairs $PAIRS --iters 3 --records 16777216
done; done; done
echo "== LSU dst"; LLAMA_LSU_SEGS=1 python tools/profile_pairs.py --config C3 --pairs aos:soa_mb,aos_aligned:soa_mb,soa_mb:aos --iters 3 --records 16777216
