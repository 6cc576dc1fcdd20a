# Listing-1 (21-byte packed records, 1- to 8-byte leaves): every pair of the
# plain kinds at 16M records, default plan vs the JIT permute forced (jit=2)
K="aos aos_aligned soa_mb soa_sb aosoa8 aosoa32"
P=""
for a in $K; do for b in $K; do [ $a != $b ] && P="$P,$a:$b"; done; done
P=${P#,}
echo "== default"; python tools/profile_pairs.py --config C4 --records 16777216 --pairs $P --iters 5 | sed 's/{.*jit.: \(True\|False\)}/jit=\1/'
echo "== jit=2"; python tools/profile_pairs.py --config C4 --records 16777216 --pairs $P --iters 5 --knobs jit=2 | sed 's/{.*jit.: \(True\|False\)}/jit=\1/'
