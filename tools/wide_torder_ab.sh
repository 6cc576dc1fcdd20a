for c in "hep100 1024 soa_mb/col aos/row" "hep100 1024 soa_mb/col aos_aligned/row" "hep100 1024 aos/row soa_mb/col" "hep100 1024 soa_mb/row soa_mb/col" "hep100 1024 soa_sb/col aos/morton" "hep100 1024 aos/morton soa_mb/col"; do
  for k in wide_torder=0 wide_torder=1; do python tools/wide_once.py $c $k | grep GB/s | sed "s|^|$k |"; done
done
