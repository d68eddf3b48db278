mkdir -p gpurun_out
HEGRID_TC_TIMING=1 timeout 600 python tools/e2e_probe.py cfg4 > gpurun_out/e2e.log 2>&1
echo done
