for v in base d1 d2 d3; do
  if [ $v = base ]; then unset HEGRID_LIB; else export HEGRID_LIB=tmp_libs/lib_$v.so; fi
  timeout 300 python bench.py --no-cpu --no-e2e --steps 10 --warmup 3 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', d['ms_per_step'], d['roofline']['frac'])"
done
