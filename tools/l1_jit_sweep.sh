# JIT permute geometry on the Listing-1 AoS pairs (16M records)
P=aos:soa_mb,soa_mb:aos,aos:aos_aligned,aos_aligned:aos,aos:aosoa8,aosoa32:aos,aos_aligned:soa_mb,soa_mb:aos_aligned,aos_aligned:aosoa32,aosoa8:aos_aligned,aos:soa_sb,soa_sb:aos
for k in "" jit_tile=256 jit_tile=128 jit_stages=2 jit_stages=4 jit_soa_tma=0 jit_soa_tma=2 jit_dst_bufs=2 jit_tile=256,jit_stages=4; do
  echo "== $k"; timeout 300 python tools/profile_pairs.py --config C4 --records 16777216 --pairs $P --knobs "$k" --iters 5 | sed 's/{.*jit.: \(True\|False\)}/jit=\1/'
done
