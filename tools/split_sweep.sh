#!/bin/bash
# cfg3: the split-tile factor (HEGRID_TC_SPLIT) vs device-resident ms/step
for k in 4 5 7 10 12 14 16; do
  r=$(HEGRID_TC_SPLIT=$k timeout 300 python bench.py --no-cpu --no-e2e --steps 5 --warmup 3 --workload cfg3 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step'],3))")
  echo "split $k $r"
done
