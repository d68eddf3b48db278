#!/bin/bash
# One GPU session producing the round's evidence under gpurun_out/ (copied to profiles/rNN by
# hand): GPU tests, smoke, ncu DRAM traffic of the top kernel (fed to bench.py's roofline
# line), the bench line (N=1 default) and cfg2/cfg3 lines, the ncu launch list of the bench
# command, one ncu --set full capture of the top kernel, the cfg5 streamed run.
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,clocks.mem --format=csv > gpurun_out/smi.txt
lscpu | grep -E "Model name|^CPU\(s\)" > gpurun_out/cpu.txt
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1
timeout 300 python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1
timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:k_accum -s 1 -c 1 --csv --log-file gpurun_out/traffic.csv python tools/profile_run.py --workload cfg4 --engine tc --launches 2 > gpurun_out/ncu_traffic.log 2>&1
python tools/traffic_json.py gpurun_out/traffic.csv cfg4 > gpurun_out/ncu_traffic.json && cp gpurun_out/ncu_traffic.json profiles/ncu_traffic.json
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
for wl in cfg2 cfg3; do timeout 600 python bench.py --workload $wl --no-cpu --no-e2e > gpurun_out/bench_$wl.json 2>> gpurun_out/bench.err; done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 --no-cpu --no-e2e > gpurun_out/bench_ncu.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_accum -s 1 -c 1 -o gpurun_out/prof_full python tools/profile_run.py --workload cfg4 --engine tc --launches 2 > gpurun_out/ncu_full.log 2>&1
CFG5_POOL=2 timeout 900 python tools/cfg5_stream.py > gpurun_out/cfg5.json 2> gpurun_out/cfg5.err
echo done
