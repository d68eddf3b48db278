for v in base named; do
  if [ $v = base ]; then unset HEGRID_LIB; else export HEGRID_LIB=tmp_libs/lib_$v.so; fi
  timeout 300 python bench.py --no-cpu --no-e2e --steps 10 --warmup 3 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v cfg4', d['ms_per_step'], d['roofline']['frac'])"
  timeout 300 python bench.py --workload cfg3 --no-cpu --no-e2e --steps 5 --warmup 3 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v cfg3', d['ms_per_step'])"
done
HEGRID_LIB=tmp_libs/lib_named.so timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "tc" 2>&1 | tail -2
