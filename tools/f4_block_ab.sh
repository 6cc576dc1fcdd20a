# A/B: block programs (knob jit_block) for SoA sources into AoS destinations (Particle7 4096^2), 3 rounds
for r in 1 2 3; do
for c in "particle7 4096 soa_mb/morton aos/col" "particle7 4096 soa_mb/row aos/col" "particle7 4096 soa_mb/col aos/row" "particle7 4096 soa_mb/morton aos/row"; do
  for k in jit_block=0 jit_block=1; do python tools/wide_once.py $c $k | grep GB/s | sed "s|^|$k $c: |"; done
done; done
