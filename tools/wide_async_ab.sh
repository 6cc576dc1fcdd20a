# A/B of cp.async element copies in the wide kernel's element-wise -> AoS mode (knob wide_async), interleaved
for r in 1 2 3; do
for c in "hep100 1024 soa_mb/col aos/row" "hep100 1024 soa_mb/col aos_aligned/row" "hep100 1024 soa_sb/row aos_aligned/col" "hep100 2048 soa_mb/col aos/row" "hep100 1024 aosoa8/morton aos_aligned/row"; do
  for k in wide_async=0 wide_async=1; do python tools/wide_once.py $c $k | grep GB/s | sed "s|^|$k $c: |"; done
done; done
