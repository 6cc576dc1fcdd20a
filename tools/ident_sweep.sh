P=aos:aos,soa_mb:soa_mb,aosoa8:aosoa8,aosoa32:aosoa32
python tools/profile_pairs.py --config C2 --pairs $P --iters 10 | sed 's/{.*}//'
for k in "" bulk_chunk=131072 bulk_chunk=32768 bulk_stages=4 bulk_stages=2 blobcopy_lsu=1; do echo "== blobcopy $k"; python tools/profile_pairs.py --config C2 --pairs $P --iters 10 --path blobcopy --knobs "$k" | sed 's/{.*}//'; done
python tools/profile_pairs.py --config C2 --pairs soa_sb:soa_sb --iters 10 | sed 's/{.*}//'
python tools/profile_pairs.py --config C2 --pairs soa_sb:soa_sb --iters 10 --path blobcopy | sed 's/{.*}//'
