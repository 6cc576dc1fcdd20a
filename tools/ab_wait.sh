VARIANTS="old new" bash tools/ab_c2.sh > gpurun_out/ab.log 2>&1
for v in old new; do
  case $v in old) R=tools/ab_old;; *) R=;; esac
  echo "== $v"
  LLAMA_PKG_ROOT=$R python tools/split_ab.py aos:split_mb_a8,aos:split_mb_a32,soa_mb:split_mb_a8 | awk '{print $1, $3, $(NF-3), $(NF-1)}'
  LLAMA_PKG_ROOT=$R python tools/profile_pairs.py --config C4 --pairs aosoa32:soa_sb --iters 5 | awk '{print $1, $3, $(NF-3), $(NF-1)}'
  LLAMA_PKG_ROOT=$R python tools/profile_pairs.py --config C3 --records 8388608 --pairs aos:aos_aligned,soa_mb:aos --iters 3 | awk '{print $1, $3, $(NF-3), $(NF-1)}'
done > gpurun_out/ab2.log 2>&1
