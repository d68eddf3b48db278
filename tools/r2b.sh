mkdir -p gpurun_out
timeout 120 python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1; echo smoke rc=$? >> gpurun_out/smoke.log
timeout 300 python bench.py --no-cpu --no-e2e --steps 5 > gpurun_out/b4_v2.json 2> gpurun_out/b.err
HEGRID_TC_V1=1 timeout 300 python bench.py --no-cpu --no-e2e --steps 5 > gpurun_out/b4_v1.json 2>> gpurun_out/b.err
for wl in cfg2 cfg3; do timeout 300 python bench.py --workload $wl --no-cpu --no-e2e --steps 5 > gpurun_out/b_$wl.json 2>>gpurun_out/b.err; done
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1
echo done
