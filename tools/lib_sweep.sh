#!/bin/bash
# short cfg4 bench (device-resident) for each experiment library: tools/lib_sweep.sh NAME...
for v in "$@"; do
  if [ "$v" = base ]; then unset HEGRID_LIB; else export HEGRID_LIB=tmp_libs/lib_$v.so; fi
  r=$(timeout 300 python bench.py --no-cpu --no-e2e --steps 5 --warmup 3 ${BENCH_ARGS} 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step'],3))" 2>&1 | tail -1)
  echo "$v $r"
done
