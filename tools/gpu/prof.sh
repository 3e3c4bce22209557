set -e
CMD="python bench.py --envs 512 --steps 1 --warmup 1 --no-e2e --no-cpu"
$CMD > gpurun_out/b512.json 2> gpurun_out/b512.err
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r1.csv $CMD > /dev/null 2>&1
for k in ${KERNELS:-sort_bin_kernel project_kernel}; do
  ncu --set full --clock-control none --import-source on -k regex:$k -s 1 -c 1 -o gpurun_out/prof_$k $CMD > gpurun_out/ncu_$k.log 2>&1 || echo "ncu $k failed"
done
