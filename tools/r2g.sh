mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_sanitizer.py tests/test_gpu_multi.py -q > gpurun_out/pytest_san.log 2>&1
bash tools/racecheck_tc.sh
timeout 600 python tools/e2e_probe.py cfg4 > gpurun_out/e2e.log 2>&1
echo done
