#!/bin/bash
# Per-pair sweep of every config family for profiles/ (run after profile_round.sh).
echo "### C2 (16M Particle7)"
python tools/profile_pairs.py --pairs aos:aos,aos:soa_mb,aos:aosoa8,aos:aosoa32,soa_mb:aos,soa_mb:soa_mb,soa_mb:aosoa8,soa_mb:aosoa32,aosoa8:aos,aosoa8:soa_mb,aosoa8:aosoa8,aosoa8:aosoa32,aosoa32:aos,aosoa32:soa_mb,aosoa32:aosoa8,aosoa32:aosoa32 --iters 10
echo "### C3 (HEP100, 16M-record prefix)"
python tools/profile_pairs.py --config C3 --records 16777216 --pairs aos:aos_aligned,aos_aligned:aos,aos:soa_mb,soa_mb:aos,aos_aligned:soa_mb,soa_mb:aos_aligned,soa_mb:soa_mb --iters 3
echo "### C4 (Listing1 8192x8192)"
python tools/profile_pairs.py --config C4 --pairs aosoa32:soa_sb --iters 5
echo "### f1 splits"
python tools/split_ab.py
python tools/profile_pairs.py --config C4 --records 67108864 --pairs aos:split_pos,split_pos:aos,aos_aligned:split_pos,split_pos:soa_sb --iters 3
python tools/profile_pairs.py --config C3 --records 8388608 --pairs aos:split_hep,split_hep:aos,soa_mb:split_hep,split_hep:soa_mb --iters 3
echo "### f4 linearisations / tracing"
python tools/f4_bench.py
