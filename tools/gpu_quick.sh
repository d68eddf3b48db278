mkdir -p gpurun_out
timeout 300 python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_pairs.py tests/test_gpu_fullsize.py -m gpu -q -x > gpurun_out/pytest_q.log 2>&1
timeout 300 python bench.py --no-cpu --no-e2e --steps 5 > gpurun_out/b4.json 2> gpurun_out/b.err
for wl in cfg2 cfg3; do timeout 300 python bench.py --workload $wl --no-cpu --no-e2e --steps 5 > gpurun_out/b_$wl.json 2>>gpurun_out/b.err; done
echo done
