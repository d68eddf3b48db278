mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1
tail -3 gpurun_out/pytest_gpu.log
timeout 300 python bench.py --no-cpu --no-e2e --steps 10 --warmup 3 > gpurun_out/bench_q.json 2>gpurun_out/bench_q.err
tail -1 gpurun_out/bench_q.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['value'], d['roofline']['frac'], d['alu_view']['frac'])"
