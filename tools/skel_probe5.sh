#!/bin/bash
export HEGRID_TC_PW=1
for x in "prof 10026" "prof 8224"; do set -- $x
  echo "== $1 dbg=$2"
  HEGRID_LIB=tmp_libs/lib_$1.so HEGRID_TC_DEBUG=$2 timeout 120 python tools/profile_run.py --workload cfg4 --channels 1024 --engine tc --launches 1 2>&1 | grep "tc " | grep -v "max chunks" | head -44
done
