K=${K:-raster_warp_kernel}
SMALL="python bench.py --envs 512 --steps 1 --warmup 3 --no-e2e --no-cpu"
$SMALL > gpurun_out/small_plain.json 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:$K -s 1 -c 1 -o gpurun_out/full_$K $SMALL > gpurun_out/ncu_$K.log 2>&1; tail -2 gpurun_out/ncu_$K.log
