#!/bin/bash
python tools/profile_pairs.py --pairs aos:aos,soa_mb:soa_mb,aos:soa_mb,soa_mb:aos,aos:aosoa8,soa_mb:aosoa8,aosoa8:aosoa32 --iters 10
python tools/profile_pairs.py --config C4 --pairs aosoa32:soa_sb --iters 10
python tools/profile_pairs.py --config C4 --pairs aosoa32:soa_sb --iters 10 --path run
for tb in 0 32768 65536; do for bud in 75000 120000; do
  echo "== C3 TILE=$tb BUDGET=$bud"
  if [ $tb -eq 0 ]; then
    python tools/profile_pairs.py --config C3 --pairs aos:aos_aligned,aos_aligned:aos,aos:soa_mb,soa_mb:aos,aos_aligned:soa_mb,soa_mb:aos_aligned --iters 3
  else
    LLAMA_TILE_BYTES=$tb LLAMA_SMEM_BUDGET=$bud python tools/profile_pairs.py --config C3 --pairs aos:aos_aligned,aos_aligned:aos,aos:soa_mb,soa_mb:aos,aos_aligned:soa_mb,soa_mb:aos_aligned --iters 3
  fi
done; done
