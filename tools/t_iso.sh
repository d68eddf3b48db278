timeout 300 python -m pytest tests/test_gpu_parity.py -q -x 2>&1 | tail -1
for m in "0 16" "1 8"; do set -- $m; HEGRID_TC_DENSE=$1 HEGRID_TC_PROMOTE=$2 timeout 120 python tools/det_small.py sparse 2>&1 | tail -1; done
timeout 120 python tools/det_small.py dense 2>&1 | tail -1
timeout 300 python tools/diag_tc_dense.py 2>&1 | grep -E "^tc|^simt"
timeout 800 python tools/err_report.py cfg2 cfg4
bash tools/tc_ablate.sh 2>&1 | grep dbg | head -2
