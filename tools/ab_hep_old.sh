P=soa_mb:aos_aligned,aos:soa_mb,aos_aligned:soa_mb
for rep in 1 2; do for v in old new; do R=; [ $v = old ] && R=tools/ab_old; echo "== $v"; LLAMA_PKG_ROOT=$R python tools/profile_pairs.py --config C3 --records 8388608 --pairs $P --iters 3 | awk '{print $1, $3, $(NF-3), $(NF-1)}'; done; done
