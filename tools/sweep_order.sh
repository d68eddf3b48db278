mkdir -p gpurun_out
for env in "X=1" "HEGRID_TC_SNAKE=1" "HEGRID_TC_SUPER=2" "HEGRID_TC_SUPER=2 HEGRID_TC_SNAKE=1" "HEGRID_TC_GROUP=16" "HEGRID_TC_GROUP=8 HEGRID_TC_SUPER=2 HEGRID_TC_SNAKE=1" "HEGRID_TC_GROUP=4 HEGRID_TC_SNAKE=1"; do
  echo "== $env"; env $env timeout 300 python bench.py --no-cpu --no-e2e --steps 5 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d['ms_per_step'],3))"
done
