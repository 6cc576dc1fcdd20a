# A/B of the wide kernel's tensor-map TMA images (knob wide_tma), interleaved, 3 rounds
for r in 1 2 3; do
for c in "hep100 1024 aos/row soa_mb/col" "hep100 1024 soa_mb/col aos/row" "hep100 1024 aos/col soa_sb/row" "hep100 1024 soa_sb/row aos_aligned/col" "hep100 1024 aos/row aos/col" "hep100 2048 aos/row soa_mb/col" "hep100 2048 soa_mb/col aos/row"; do
  for k in wide_tma=0 wide_tma=1; do python tools/wide_once.py $c $k | grep GB/s | sed "s|^|$k $c: |"; done
done; done
