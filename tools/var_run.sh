#!/bin/bash
# run the determinism checks, profile counters and a short bench for each variant lib given
for v in "$@"; do
  if [ "$v" = base ]; then unset HEGRID_LIB; else export HEGRID_LIB=tmp_libs/lib_$v.so; fi
  echo "== $v"
  for m in "0 16" "1 8" "1 4"; do set -- $m; HEGRID_TC_DENSE=$1 HEGRID_TC_PROMOTE=$2 timeout 120 python tools/det_small.py sparse 2>&1 | tail -1; done
  HEGRID_TC_DENSE=1 timeout 120 python tools/det_small.py dense 2>&1 | tail -1
  HEGRID_TC_DEBUG=32 timeout 120 python tools/profile_run.py --workload cfg4 --channels 1024 --engine tc --launches 1 2>&1 | grep "tc prof" | head -1
  timeout 300 python bench.py --no-cpu --no-e2e --steps 5 --warmup 3 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'])"
done
