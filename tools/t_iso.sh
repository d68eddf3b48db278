timeout 300 python -m pytest tests/test_gpu_parity.py -q -x 2>&1 | tail -1
t=$(python bench.py --steps 5 --warmup 3 --no-cpu --no-e2e --engine tc 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d["ms_per_step"],2))')
echo "prod $t ms"
export HEGRID_LIB=tmp_libs/lib_prof.so
t=$(python bench.py --steps 5 --warmup 3 --no-cpu --no-e2e --engine tc 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d["ms_per_step"],2))')
echo "prof-build $t ms"
