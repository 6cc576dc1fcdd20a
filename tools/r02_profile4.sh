#!/bin/bash
# ncu traffic of the transposing-copy bench sub-configs (F4_p7, F4_hep), pair
# by pair in bench.py's order (profiles/traffic.json via tools/traffic_from_ncu.py
# "csv:@CONFIG"), each command first run without ncu.
set -x
mkdir -p gpurun_out
M="gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum"
pairs() { python -c "import bench; print(','.join(a+':'+b for a,b in bench.pairs_of('$1')))"; }
for c in F4_p7 F4_hep; do
  P=$(pairs $c)
  python tools/profile_pairs.py --subcfg $c --iters 1 --pairs $P > gpurun_out/r02_pp_$c.txt 2>&1 || exit 1
  ncu --metrics $M --clock-control none --csv --log-file gpurun_out/r02_traffic3_$c.csv \
    python tools/profile_pairs.py --subcfg $c --iters 1 --pairs $P > /dev/null 2>&1
done
ls -la gpurun_out/r02_traffic3_F4*
