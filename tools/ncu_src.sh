#!/bin/bash
# ncu source-level capture of one k_accum_tc launch (cfg4, 1024 channels)
mkdir -p gpurun_out
timeout 300 ncu --set full --clock-control none --import-source on -k regex:k_accum_tc -s 1 -c 1 -o gpurun_out/${1:-prof_src} python tools/profile_run.py --workload cfg4 --channels 1024 --engine tc --launches 2 > gpurun_out/ncu_src.log 2>&1
tail -2 gpurun_out/ncu_src.log
