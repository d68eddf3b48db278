#!/bin/bash
# per-A-warp lag (g_tla a_full times of chunk 44) for prof builds: tools/lag_probe.sh LIB...
export HEGRID_TC_PW=1
for lib in "$@"; do for d in 10026 8224; do
  echo "== $lib dbg=$d"
  HEGRID_LIB=tmp_libs/lib_$lib.so HEGRID_TC_DEBUG=$d timeout 120 python tools/profile_run.py --workload cfg4 --channels 1024 --engine tc --launches 1 2>&1 | grep "tc prof\|tla.*4[4-5] afull" | cut -c1-120
done; done
