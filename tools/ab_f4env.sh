for rep in 1 2; do
for e in "LLAMA_TRANSPOSE_RAW1=0" "LLAMA_TRANSPOSE_RAW1=1"; do
  echo "== $e"; env $e python tools/f4_bench.py 2>&1 | grep transpose | awk '{print $2, $4, $(NF-3), $(NF-1)}'
done; done
