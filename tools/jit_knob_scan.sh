# knob variants of the JIT permute over the bench's JIT pairs (C3 at 16M records, C4_pairs / F1 at the
# bench sizes): which pair gains > 3% from which variant
pairs() { python -c "import bench; print(','.join(a+':'+b for a,b in bench.pairs_of('$1')))"; }
for c in "C3 C3 16777216" "C3_soa_sb C3 16777216" "C4_pairs C4 67108864" "F1_hep C3 16777216" "F1_listing1 C4 67108864"; do
  set -- $c
  for k in "" "jit_tile=128" "jit_tile=256" "jit_tile=512" "jit_dst_bufs=2" "jit_ctas=3" "jit_ctas=5" "jit_stages=4" "jit_soa_tma=0" "jit_soa_tma=2" "jit_group=2"; do
    python tools/profile_pairs.py --config $2 --records $3 --iters 10 --pairs $(pairs $1) --knobs "$k" 2>&1 | grep " ms " | sed "s|^|$1 [$k] |"
  done
done
