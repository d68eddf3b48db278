#!/bin/bash
# time the TC kernel with parts disabled (HEGRID_TC_DEBUG bits: 1 = no B work, 2 = no MMAs, 4 = no V loads)
for d in 0 1 2 4 3 5 6 7; do
  echo "dbg=$d $(HEGRID_TC_DEBUG=$d python bench.py --steps 3 --warmup 2 --no-cpu --no-e2e --engine tc | python -c 'import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d["ms_per_step"],2))')"
done
