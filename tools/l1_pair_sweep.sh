# knob sweep of the weakest layout-copy pair of the bench line: Listing-1
# packed AoS -> aligned AoS, 64M records (C4_pairs), through the JIT permute
P="aos:aos_aligned"
for k in "" "jit_tile=256" "jit_tile=1024" "jit_stages=2" "jit_stages=4" "jit_dst_bufs=2" "jit_dst_bufs=4" \
         "jit_ctas=3" "jit_ctas=1" "jit_pad=0" "jit_group=1" "jit_group=2" "jit_tile=1024,jit_stages=2" \
         "jit_tile=256,jit_ctas=3" "jit_tile=256,jit_stages=4,jit_dst_bufs=4" "jit=0" "word_mode=0,jit=0"; do
  python tools/profile_pairs.py --config C4 --records 67108864 --iters 20 --pairs $P --knobs "$k" 2>&1 | tail -1 | sed "s|^|[$k] |"
done
