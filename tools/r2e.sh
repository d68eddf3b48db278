mkdir -p gpurun_out
HEGRID_LIB=tmp_libs/lib_prof.so HEGRID_TC_DEBUG=32 timeout 300 python tools/profile_run.py --workload cfg4 --launches 1 > gpurun_out/prof.log 2>&1
timeout 300 python bench.py --no-cpu --no-e2e --steps 5 > gpurun_out/b4_v2.json 2> gpurun_out/b.err
for wl in cfg2 cfg3; do timeout 300 python bench.py --workload $wl --no-cpu --no-e2e --steps 5 > gpurun_out/b_$wl.json 2>>gpurun_out/b.err; done
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_pairs.py -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1
echo done
