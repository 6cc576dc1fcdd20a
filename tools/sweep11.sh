#!/bin/bash
for tb in 32768 49152 65536; do for bud in 75000 120000 230000; do for st in 2 3 4; do
  echo "== TB=$tb BUD=$bud ST=$st"
  LLAMA_TILE_BYTES=$tb LLAMA_SMEM_BUDGET=$bud LLAMA_STAGES=$st python tools/profile_pairs.py --pairs aos:soa_mb,aos:aosoa8,aosoa8:aosoa32,soa_mb:aosoa32 --iters 10
done; done; done
for tb in 16384 32768 65536; do for bud in 75000 120000; do for st in 2 3 4; do
  echo "== C3 TB=$tb BUD=$bud ST=$st"
  LLAMA_TILE_BYTES=$tb LLAMA_SMEM_BUDGET=$bud LLAMA_STAGES=$st python tools/profile_pairs.py --config C3 --records 16777216 --pairs aos:aos_aligned,aos:soa_mb,aos_aligned:soa_mb --iters 3
done; done; done
