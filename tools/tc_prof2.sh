#!/bin/bash
for d in 32 96 160 226; do
  echo "== dbg=$d"; HEGRID_TC_DEBUG=$d timeout 120 python tools/profile_run.py --workload cfg4 --channels 1024 --engine tc --launches 1 2>&1 | grep "tc prof"
done
