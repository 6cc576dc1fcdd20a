# A/B of the pipelined E -> E path of the wide kernel (knob wide_pipe), interleaved, 3 rounds
for r in 1 2 3; do
for c in "hep100 1024 soa_mb/row soa_mb/col" "hep100 1024 soa_sb/col soa_mb/morton" "hep100 1024 soa_mb/col soa_sb/row" "hep100 2048 soa_mb/row soa_sb/col" "hep100 1024 aosoa8/col soa_mb/row"; do
  for k in wide_pipe=0 wide_pipe=1; do python tools/wide_once.py $c $k | grep GB/s | sed "s|^|$k $c: |"; done
done; done
