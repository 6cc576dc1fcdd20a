set -x
P="--iters 5"
python tools/profile_pairs.py --config C3 --records 8388608 $P --pairs soa_mb:split_hep,split_hep:soa_mb,aos:split_hep,split_hep:aos,aos_aligned:split_hep > gpurun_out/split.txt 2>&1
python tools/profile_pairs.py --config C3 --records 8388608 $P --knobs jit=0 --pairs soa_mb:split_hep,split_hep:soa_mb,aos:split_hep,split_hep:aos,aos_aligned:split_hep >> gpurun_out/split.txt 2>&1
python tools/profile_pairs.py --config C4 --records 67108864 $P --pairs aos_aligned:split_pos,aos:split_pos,split_pos:aos,soa_mb:split_pos >> gpurun_out/split.txt 2>&1
python tools/profile_pairs.py --config C4 --records 67108864 $P --knobs jit=0 --pairs aos_aligned:split_pos,aos:split_pos,split_pos:aos,soa_mb:split_pos >> gpurun_out/split.txt 2>&1
python tools/profile_pairs.py --config C2 $P --pairs aos:split_p7,split_p7:aos,soa_mb:split_p7,split_p7:soa_mb,aosoa8:split_p7 >> gpurun_out/split.txt 2>&1
python tools/profile_pairs.py --config C2 $P --knobs jit=0 --pairs aos:split_p7,split_p7:aos,soa_mb:split_p7,split_p7:soa_mb,aosoa8:split_p7 >> gpurun_out/split.txt 2>&1
python tools/profile_pairs.py --config C2 $P --knobs jit=2 --pairs aos:soa_mb,soa_mb:aos,aos:aosoa8,aosoa32:soa_mb >> gpurun_out/split.txt 2>&1
python tools/profile_pairs.py --config C4 --records 67108864 $P --knobs jit=2 --pairs aosoa32:soa_sb,aos:soa_mb,soa_mb:aos >> gpurun_out/split.txt 2>&1
python tools/profile_pairs.py --config C3 --records 16777216 --iters 1 --pairs soa_mb:aos,aos:soa_mb > /dev/null 2>&1 || exit 1
ncu --set full --clock-control none --import-source on -k regex:llb_jit -c 2 -o gpurun_out/jit_full python tools/profile_pairs.py --config C3 --records 16777216 --iters 1 --pairs soa_mb:aos,aos:soa_mb > gpurun_out/ncu_jit.log 2>&1
cat gpurun_out/split.txt | grep -v "^+"
