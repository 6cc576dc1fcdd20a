# JIT permute record-group sweep on HEP100 (16M records) and Listing-1 splits
P=aos:soa_mb,soa_mb:aos,aos:aos_aligned,aos_aligned:soa_mb,soa_mb:aos_aligned,aos_aligned:aos
for k in "" jit_group=2 jit_group=4 jit_group=4,jit_stages=2,jit_dst_bufs=2 jit_group=2,jit_tile=128; do
  echo "== $k"; timeout 300 python tools/profile_pairs.py --config C3 --records 16777216 --pairs $P --knobs "$k" --iters 5 | sed 's/{.*jit.: True}//'
done
