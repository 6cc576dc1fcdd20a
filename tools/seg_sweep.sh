# SoA SB <-> MB: the per-leaf bulk copy (path blobcopy) vs the tile permute / JIT program
for c in "C2 16777216" "C4 16777216" "C3 4194304"; do set -- $c
  for pth in "" "--path blobcopy" "--path permute"; do echo "== $1 $2 $pth"; python tools/profile_pairs.py --config $1 --records $2 --pairs soa_sb:soa_mb,soa_mb:soa_sb,soa_sb:soa_sb --iters 20 $pth | sed 's/{.*}//'; done
done
