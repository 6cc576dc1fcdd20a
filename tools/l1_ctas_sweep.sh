# JIT permute: CTAs per SM (launch bounds) x tile on Listing-1 pairs (16M) and HEP100 pairs (16M)
P=aos:soa_mb,soa_mb:aos,aos:aos_aligned,aos_aligned:aos,aos:aosoa8,aosoa32:aos,soa_sb:aos,aos_aligned:split_pos,soa_mb:split_pos,split_pos:aos
for k in "" jit_ctas=5 jit_ctas=6 jit_ctas=6,jit_tile=128 jit_ctas=5,jit_tile=512; do
  echo "== $k"; timeout 300 python tools/profile_pairs.py --config C4 --records 16777216 --pairs $P --knobs "$k" --iters 20 | sed 's/{.*jit.: \(True\|False\)}/jit=\1/'
done
