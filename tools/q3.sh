timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "tc" 2>&1 | tail -2
HEGRID_TC_PW=1 timeout 300 python bench.py --no-cpu --no-e2e --steps 10 --warmup 3 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('pw=1', d['ms_per_step'], d['roofline']['frac'])"
