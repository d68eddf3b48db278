#!/bin/bash
# CTA walk vs DRAM traffic of k_accum_tc (cfg4): GROUP = channel blocks adjacent per tile,
# SUPER = S x S super-tiles, SNAKE = odd tile rows walk their entries backwards
for cfg in ${ORDERS:-"32 1 0" "32 3 0" "8 2 0" "32 1 1" "8 3 1" "4 4 1" "2 4 1" "1 1 0" "1 3 1"}; do
  set -- $cfg
  export HEGRID_TC_GROUP=$1 HEGRID_TC_SUPER=$2 HEGRID_TC_SNAKE=$3
  timeout 300 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:k_accum -s 1 -c 1 --csv --log-file /tmp/tr.csv python tools/profile_run.py --workload cfg4 --engine tc --launches 2 > /dev/null 2>&1
  python tools/traffic_json.py /tmp/tr.csv cfg4 | python -c "import json,sys; d=json.load(sys.stdin)['cfg4']; print('group $1 super $2 snake $3: %.2f GB, %.2f ms under ncu' % (d['dram_bytes_per_launch']/1e9, d['duration_ns_under_ncu']/1e6))"
done
