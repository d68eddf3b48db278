#!/bin/bash
# quick TC check: parity, determinism, profile counters, short bench
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "tc or TC" 2>&1 | tail -3
for m in "0 16" "1 8"; do set -- $m; HEGRID_TC_DENSE=$1 HEGRID_TC_PROMOTE=$2 timeout 120 python tools/det_small.py sparse 2>&1 | tail -1; done
HEGRID_TC_DENSE=1 timeout 120 python tools/det_small.py dense 2>&1 | tail -1
HEGRID_TC_DEBUG=32 timeout 120 python tools/profile_run.py --workload cfg4 --channels 1024 --engine tc --launches 1 2>&1 | grep "tc prof"
timeout 300 python bench.py --no-cpu --no-e2e --steps 5 --warmup 3 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['value'], d['roofline'])"
