#!/bin/bash
# f4 transposes: two environment variants of the working tree, alternating (A_ENV / B_ENV).
for rep in 1 2; do
for e in "${A_ENV:-X=0}" "${B_ENV:-X=1}"; do
  echo "== $e"; env $e python tools/f4_bench.py 2>&1 | grep transpose | awk '{print $2, $4, $(NF-3), $(NF-1)}'
done; done
