mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,clocks.mem --format=csv > gpurun_out/smi.txt
lscpu | grep -E "Model name|^CPU\(s\)" > gpurun_out/cpu.txt
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1
timeout 600 python bench.py --no-cpu > gpurun_out/bench.json 2> gpurun_out/bench.err
for wl in cfg2 cfg3; do timeout 300 python bench.py --workload $wl --no-cpu --no-e2e > gpurun_out/bench_$wl.json 2>>gpurun_out/bench.err; done
echo done
