# racecheck reports of the tensor-core kernels (recorded, see tests/test_gpu_sanitizer.py)
mkdir -p gpurun_out
for m in tc_otf tc_pw; do
  /usr/local/cuda/bin/compute-sanitizer --tool racecheck --print-limit 200 python tools/sanitize_case.py $m > gpurun_out/racecheck_$m.log 2>&1
done
