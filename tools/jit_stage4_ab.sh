# A/B: 4 source stages for packed (misaligned) HEP100 AoS into all-SoA destinations (16M records), 3 rounds
for r in 1 2 3; do
  for k in "jit_stages=3" ""; do
    python tools/profile_pairs.py --config C3 --records 16777216 --iters 10 --pairs aos:soa_mb,aos:soa_sb,aos_aligned:soa_mb --knobs "$k" 2>&1 | grep " ms " | sed "s|^|[$k] |"
  done
done
