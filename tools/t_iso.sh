timeout 300 python -m pytest tests/test_gpu_parity.py -q -x 2>&1 | tail -1
for d in 0 3; do
  t=$(HEGRID_TC_DEBUG=$d python bench.py --steps 3 --warmup 2 --no-cpu --no-e2e --engine tc 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d["ms_per_step"],2))')
  p=$(HEGRID_TC_DEBUG=$((d+32)) timeout 120 python tools/profile_run.py --workload cfg4 --channels 1024 --engine tc --launches 1 2>&1 | grep "tc prof" | head -1| cut -c1-400)
  echo "dbg=$d $t ms | $p"
done
