for d in 32768 0; do
  echo "== dbg $d"
  HEGRID_TC_DEBUG=$d HEGRID_TC_DENSE=0 timeout 120 python tools/det_small.py sparse 2>&1 | tail -1
  HEGRID_TC_DEBUG=$d HEGRID_TC_DENSE=0 timeout 120 python tools/det_small.py sparse 2>&1 | tail -1
done
