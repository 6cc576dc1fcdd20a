# knob sweep of the Listing-1 split pairs (64M records, bench F1_listing1)
P=aos:split_pos,split_pos:aos_aligned,soa_mb:split_pos,split_pos:aos,aos_aligned:split_pos,split_pos:soa_mb
for k in "" jit_tile=256 jit_tile=256,jit_stages=4 jit_tile=256,jit_stages=2 "" jit_tile=256; do
  echo "== $k"; timeout 300 python tools/profile_pairs.py --config C4 --records 67108864 --pairs $P --knobs "$k" --iters 5 | sed 's/{.*jit.: True}//'
done
