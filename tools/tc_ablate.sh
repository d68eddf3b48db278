#!/bin/bash
# needs the profiling build: tools/build_variant.sh prof -DHG_TC_PROF
export HEGRID_LIB=${HEGRID_LIB:-tmp_libs/lib_prof.so}
# time the TC kernel with parts disabled (HEGRID_TC_DEBUG bits: 1 = no B work, 2 = no MMAs,
# 4 = no A values, 8 = no V copies, 64 = trivial weights) and print the profile split
for d in 0 1 2 64 3 9; do
  t=$(HEGRID_TC_DEBUG=$d python bench.py --steps 3 --warmup 2 --no-cpu --no-e2e --engine tc 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d["ms_per_step"],2))')
  p=$(HEGRID_TC_DEBUG=$((d+32)) timeout 120 python tools/profile_run.py --workload cfg4 --channels 1024 --engine tc --launches 1 2>&1 | grep "tc prof" | head -1 | cut -c1-250)
  echo "dbg=$d $t ms | $p"
done
