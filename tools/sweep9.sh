#!/bin/bash
PAIRS=aos:aos_aligned,aos_aligned:aos,aos:soa_mb,soa_mb:aos,aos_aligned:soa_mb,soa_mb:aos_aligned
for lsu in 0 1; do for tb in 0 32768 49152; do
  echo "== C3 LSU=$lsu TILE=$tb"
  if [ $tb -eq 0 ]; then LLAMA_LSU_SEGS=$lsu python tools/profile_pairs.py --config C3 --pairs $PAIRS --iters 3 --records 16777216
  else LLAMA_LSU_SEGS=$lsu LLAMA_TILE_BYTES=$tb LLAMA_SMEM_BUDGET=120000 python tools/profile_pairs.py --config C3 --pairs $PAIRS --iters 3 --records 16777216; fi
done; done
echo "== C2"; python tools/profile_pairs.py --pairs aos:soa_mb,soa_mb:aos,aos:aosoa8,aos:aos_aligned,aos_aligned:aos --iters 10
echo "== C2 LSU"; LLAMA_LSU_SEGS=1 python tools/profile_pairs.py --pairs aos:soa_mb,soa_mb:aos,soa_mb:aosoa8 --iters 10
