mkdir -p gpurun_out
timeout 300 python bench.py --no-cpu --no-e2e --steps 5 > gpurun_out/b4_v2.json 2> gpurun_out/b.err
for wl in cfg2 cfg3; do timeout 300 python bench.py --workload $wl --no-cpu --no-e2e --steps 5 > gpurun_out/b_$wl.json 2>>gpurun_out/b.err; done
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1
echo done
