# Listing-1 / HEP100 AoSoA-4 pairs: default plan vs the JIT permute (jit=2), after padded blocks and misaligned elements
P=aosoa4:aos,aos:aosoa4,aos_aligned:aosoa4,aosoa4_aligned:aosoa4,aosoa4:split_pos,aosoa4_aligned:soa_mb,aosoa4_aligned:aosoa8,soa_mb:aosoa4_aligned,aosoa8:aosoa4_aligned,aosoa4_aligned:aos,split_pos:aosoa4_aligned,aosoa4:soa_mb,aosoa4:aosoa8,soa_mb:aosoa4,aosoa8:aosoa4
for k in "" jit=2 jit=2,jit_pad=0; do echo "== listing1 $k"; python tools/profile_pairs.py --config C4 --records 16777216 --pairs $P --knobs "$k" --iters 10 | sed 's/{.*jit.: \(True\|False\)}/jit=\1/'; done
H=aosoa4_aligned:soa_mb,soa_mb:aosoa4_aligned,aosoa4_aligned:aos,aos_aligned:aosoa4_aligned,soa_sb:soa_mb,soa_mb:soa_sb
for k in "" jit_pad=0 path; do
  if [ "$k" = path ]; then echo "== hep100 path=run"; python tools/profile_pairs.py --config C3 --records 4194304 --pairs soa_sb:soa_mb,soa_mb:soa_sb --path run --iters 10 | sed 's/{.*}//'; continue; fi
  echo "== hep100 $k"; python tools/profile_pairs.py --config C3 --records 4194304 --pairs $H --knobs "$k" --iters 10 | sed 's/{.*jit.: \(True\|False\)}/jit=\1/'; done
