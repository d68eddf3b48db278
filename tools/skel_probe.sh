#!/bin/bash
# per-role wait fractions and one-CTA timeline, full kernel vs hand-off skeleton (prof build)
export HEGRID_LIB=tmp_libs/lib_prof.so HEGRID_TC_PW=1
for d in 32 1834 8224 10026; do
  echo "== dbg=$d"
  HEGRID_TC_DEBUG=$d timeout 120 python tools/profile_run.py --workload cfg4 --channels 1024 --engine tc --launches 1 2>&1 | grep "tc "
done
