#!/bin/bash
PAIRS=aos:aos_aligned,aos_aligned:aos,aos:soa_mb,soa_mb:aos,aos_aligned:soa_mb,soa_mb:aos_aligned
for tb in 0 24576 49152 98304; do for dg in 0 1; do
  echo "== C3 TILE=$tb DIAG=$dg"
  if [ $tb -eq 0 ]; then LLAMA_DIAG=$dg python tools/profile_pairs.py --config C3 --pairs $PAIRS --iters 3 --records 16777216
  else LLAMA_DIAG=$dg LLAMA_TILE_BYTES=$tb LLAMA_SMEM_BUDGET=120000 python tools/profile_pairs.py --config C3 --pairs $PAIRS --iters 3 --records 16777216; fi
done; done
echo "== C4"
python tools/profile_pairs.py --config C4 --pairs aosoa32:soa_sb --iters 10
for tb in 32768 49152; do LLAMA_TILE_BYTES=$tb python tools/profile_pairs.py --config C4 --pairs aosoa32:soa_sb --iters 10; done
