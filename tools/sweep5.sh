#!/bin/bash
for ch in 16384 32768 65536; do for ns in 3 4 6 8; do
  if [ $((ch*ns)) -le 220000 ]; then
    echo "== BULK CH=$ch NS=$ns"
    LLAMA_BULK_CHUNK=$ch LLAMA_BULK_STAGES=$ns python tools/profile_pairs.py --pairs aos:aos,soa_mb:soa_mb --iters 10
  fi
done; done
echo "== LSU blobcopy"
LLAMA_BLOBCOPY_LSU=1 python tools/profile_pairs.py --pairs aos:aos,soa_mb:soa_mb --iters 10
for tb in 32768 49152 65536 98304; do for bud in 75000 120000 230000; do for st in 2 3 4; do
  echo "== PERM TILE=$tb BUDGET=$bud STAGES=$st"
  LLAMA_TILE_BYTES=$tb LLAMA_SMEM_BUDGET=$bud LLAMA_STAGES=$st python tools/profile_pairs.py --pairs aos:soa_mb,soa_mb:aos,soa_mb:aosoa8,aosoa32:soa_mb,aos:aosoa8 --iters 10
done; done; done
