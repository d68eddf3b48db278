mkdir -p gpurun_out
./tools/pipe_bench
for i in 0 1 2 3; do
ncu --set full --clock-control none -k regex:k2 -s 1 -c 1 -o gpurun_out/pb_$i ./tools/pipe_bench $i > gpurun_out/pb_ncu_$i.log 2>&1
done
