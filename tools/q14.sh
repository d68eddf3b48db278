for v in base d1 d2 d3; do
  if [ $v = base ]; then unset HEGRID_LIB; else export HEGRID_LIB=tmp_libs/lib_$v.so; fi
  HEGRID_TC_PW=1 timeout 300 python bench.py --no-cpu --no-e2e --steps 10 --warmup 3 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', d['ms_per_step'], d['roofline']['frac'])"
done
HEGRID_LIB=tmp_libs/lib_m36.so timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "tc" 2>&1 | tail -3
HEGRID_LIB=tmp_libs/lib_m36.so HEGRID_TC_PW=1 timeout 300 python tools/err_report.py cfg4 cfg2 2>&1 | tail -2
