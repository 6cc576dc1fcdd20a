# A/B of 1-d bulk copies for Morton image sides of the wide kernel (knob wide_tma), interleaved, 3 rounds
for r in 1 2 3; do
for c in "hep100 1024 aos/morton soa_mb/row" "hep100 1024 soa_mb/col aos/morton" "hep100 1024 aos_aligned/morton soa_sb/col" "hep100 1024 aos/row aos/morton" "hep100 1024 aosoa8/morton soa_mb/row"; do
  for k in wide_tma=0 wide_tma=1; do python tools/wide_once.py $c $k | grep GB/s | sed "s|^|$k $c: |"; done
done; done
