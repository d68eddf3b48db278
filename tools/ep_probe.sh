#!/bin/bash
export HEGRID_TC_PW=1
for lib in prof_ep prof_epmix; do for d in 0 1800 16384 1024 17408 512 2048; do
  r=$(HEGRID_LIB=tmp_libs/lib_$lib.so HEGRID_TC_DEBUG=$((d+32)) timeout 120 python tools/profile_run.py --workload cfg4 --channels 1024 --engine tc --launches 1 2>&1 | grep "tc prof" | grep -v "max chunks" | cut -c1-60)
  echo "$lib dbg=$d $r"
done; done
