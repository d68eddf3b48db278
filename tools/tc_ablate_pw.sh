#!/bin/bash
# PW-mode ablation with the profiling build: HEGRID_TC_DEBUG bits 2 = no MMAs, 4 = A values
# masked, 8 = no V copies; prints ms and the role split
export HEGRID_LIB=${HEGRID_LIB:-tmp_libs/lib_prof.so} HEGRID_TC_PW=1
for d in 0 2 8 10; do
  t=$(HEGRID_TC_DEBUG=$d python bench.py --steps 3 --warmup 2 --no-cpu --no-e2e --engine tc 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d["ms_per_step"],2))')
  p=$(HEGRID_TC_DEBUG=$((d+32)) timeout 120 python tools/profile_run.py --workload cfg4 --channels 1024 --engine tc --launches 1 2>&1 | grep "tc prof" | head -1 | cut -c1-330)
  echo "dbg=$d $t ms | $p"
done
