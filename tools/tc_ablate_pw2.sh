#!/bin/bash
# PW-mode ablation (profiling build): HEGRID_TC_DEBUG bits 2 = no MMAs, 8 = no V copies,
# 256 = no A value work (no split, no tcgen05.st), 512 = no weight copies, 1024 = no promotions
export HEGRID_LIB=${HEGRID_LIB:-tmp_libs/lib_prof.so} HEGRID_TC_PW=1
for d in 1802 5898 4098 2; do
  t=$(HEGRID_TC_DEBUG=$d timeout 120 python bench.py --steps 3 --warmup 2 --no-cpu --no-e2e --engine tc 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d["ms_per_step"],2))')
  p=$(HEGRID_TC_DEBUG=$((d+32)) timeout 120 python tools/profile_run.py --workload cfg4 --channels 1024 --engine tc --launches 1 2>&1 | grep "tc prof" | head -1 | cut -c1-300)
  echo "dbg=$d $t ms | $p"
done
