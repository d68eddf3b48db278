timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "tc" 2>&1 | tail -2
for pw in 1 0; do HEGRID_TC_PW=$pw timeout 300 python bench.py --no-cpu --no-e2e --steps 10 --warmup 3 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('pw=$pw', d['ms_per_step'], d['roofline']['frac'])"; done
HEGRID_TC_PW=1 HEGRID_LIB=tmp_libs/lib_prof.so HEGRID_TC_DEBUG=32 timeout 120 python tools/profile_run.py --workload cfg4 --channels 1024 --engine tc --launches 1 2>&1 | grep "tc prof" | head -1
