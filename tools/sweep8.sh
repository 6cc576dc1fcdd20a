#!/bin/bash
PAIRS=aos:aos_aligned,aos_aligned:aos,aos:soa_mb,soa_mb:aos,aos_aligned:soa_mb,soa_mb:aos_aligned
echo "== C3 default"; python tools/profile_pairs.py --config C3 --pairs $PAIRS --iters 3 --records 16777216
for tb in 32768 98304; do echo "== C3 TILE=$tb"; LLAMA_TILE_BYTES=$tb LLAMA_SMEM_BUDGET=120000 python tools/profile_pairs.py --config C3 --pairs $PAIRS --iters 3 --records 16777216; done
echo "== C2 LSU forced"; LLAMA_LSU_SEGS=1 python tools/profile_pairs.py --pairs aos:soa_mb,soa_mb:aos,soa_mb:aosoa8 --iters 10
