for v in base whalf wsplit4k wsplit2k; do
  if [ $v = base ]; then unset HEGRID_LIB; else export HEGRID_LIB=tmp_libs/lib_$v.so; fi
  HEGRID_TC_PW=1 timeout 300 python bench.py --no-cpu --no-e2e --steps 10 --warmup 3 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', d['ms_per_step'], d['roofline']['frac'])"
done
HEGRID_TC_PW=1 HEGRID_LIB=tmp_libs/lib_whalf_prof.so HEGRID_TC_DEBUG=32 timeout 120 python tools/profile_run.py --workload cfg4 --channels 1024 --engine tc --launches 1 2>&1 | grep "tc prof" | head -1
HEGRID_TC_PW=1 HEGRID_LIB=tmp_libs/lib_whalf_prof.so HEGRID_TC_DEBUG=34 timeout 120 python tools/profile_run.py --workload cfg4 --channels 1024 --engine tc --launches 1 2>&1 | grep "tc prof" | head -1
