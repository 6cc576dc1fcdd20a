#!/bin/bash
# f4 transposes: old build vs current, alternating.
for rep in 1 2; do
  for v in ${VARIANTS:-old new}; do
    case $v in old) R=tools/ab_old;; exp) R=tools/ab_exp;; *) R=;; esac
    echo "== $v"
    LLAMA_PKG_ROOT=$R python tools/f4_bench.py 2>&1 | grep transpose | awk '{print $2, $4, $(NF-3), $(NF-1)}'
  done
done
