timeout 300 python -m pytest tests/test_gpu_parity.py -q -x 2>&1 | tail -1
for m in "0 16" "1 8"; do timeout 120 python tools/det_small.py sparse 2>&1 | tail -1; done
timeout 120 python tools/det_small.py dense 2>&1 | tail -1
timeout 300 python tools/diag_tc_dense.py 2>&1 | grep -E "^tc"
timeout 800 python tools/err_report.py cfg4
t=$(python bench.py --steps 5 --warmup 3 --no-cpu --no-e2e --engine tc 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d["ms_per_step"],2))')
echo "prod $t ms"
HEGRID_LIB=tmp_libs/lib_prof.so HEGRID_TC_DEBUG=32 timeout 120 python tools/profile_run.py --workload cfg4 --channels 1024 --engine tc --launches 1 2>&1 | grep "tc prof" | head -1| cut -c1-400
