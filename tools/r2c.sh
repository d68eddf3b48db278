mkdir -p gpurun_out
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_accum_pw -s 1 -c 1 -o gpurun_out/pw_full python tools/profile_run.py --workload cfg4 --launches 2 > gpurun_out/pw_ncu.log 2>&1
echo done
