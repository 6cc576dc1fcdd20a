# A/B of the JIT permute's source stages (default: 3 while the ring fits 180 KB) against 2, over
# the bench's JIT pairs (C3 at 16M records, C4_pairs / F1 at the bench sizes), interleaved, 2 rounds
pairs() { python -c "import bench; print(','.join(a+':'+b for a,b in bench.pairs_of('$1')))"; }
for r in 1 2; do
for c in "C3 C3 16777216" "C4_pairs C4 67108864" "F1_hep C3 16777216" "F1_listing1 C4 67108864"; do
  set -- $c
  for k in "" "jit_stages=2"; do
    python tools/profile_pairs.py --config $2 --records $3 --iters 10 --pairs $(pairs $1) --knobs "$k" 2>&1 | grep " ms " | sed "s|^|$1 [$k] |"
  done
done; done
