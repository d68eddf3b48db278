#!/bin/bash
# ablations of the current kernel (prof build): cycles per CTA, cfg4 1024 channels
export HEGRID_TC_PW=1
for d in 0 2 1800 1802 4194304 256 8 512; do
  r=$(HEGRID_LIB=tmp_libs/lib_prof.so HEGRID_TC_DEBUG=$((d+32)) timeout 120 python tools/profile_run.py --workload cfg4 --channels 1024 --engine tc --launches 1 2>&1 | grep "tc prof" | grep -v "max chunks" | cut -c1-200)
  echo "dbg=$d $r"
done
