# A/B: element-wise -> AoS in 64-record tiles at 6 CTAs per SM (knob wide_ea_tile), interleaved, 3 rounds
for r in 1 2 3; do
for c in "hep100 1024 soa_mb/col aos/row" "hep100 1024 soa_mb/col aos_aligned/row" "hep100 1024 soa_sb/row aos_aligned/col" "hep100 2048 soa_mb/col aos/row" "hep100 1024 soa_mb/row aos/morton"; do
  for k in wide_ea_tile=0 wide_ea_tile=1; do python tools/wide_once.py $c $k | grep GB/s | sed "s|^|$k $c: |"; done
done; done
