timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "tc" 2>&1 | tail -2
for gs in "32 1 0" "32 1 1" "32 2 1" "16 3 1" "32 3 1" "16 4 1"; do set -- $gs
  HEGRID_TC_GROUP=$1 HEGRID_TC_SUPER=$2 HEGRID_TC_SNAKE=$3 timeout 300 python bench.py --no-cpu --no-e2e --steps 10 --warmup 3 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('group $1 super $2 snake $3', d['ms_per_step'], d['roofline']['frac'])"
done
for gs in "32 1 1" "32 2 1" "16 3 1"; do set -- $gs
  HEGRID_TC_GROUP=$1 HEGRID_TC_SUPER=$2 HEGRID_TC_SNAKE=$3 timeout 300 ncu --metrics dram__bytes_read.sum --clock-control none -k regex:k_accum -s 1 -c 1 --csv python tools/profile_run.py --workload cfg4 --engine tc --launches 2 2>/dev/null | grep dram__ | awk -F'","' -v g="$1 $2 $3" '{print g, $(NF-2), $(NF-1), $NF}'
done
