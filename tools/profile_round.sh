#!/bin/bash
# GPU-box profiling pass for one round (run under gpurun from the repo root):
#   1. the bench command without ncu (must exit 0 first)
#   2. the ncu launch list of the same command (gpu__time_duration per launch)
#   3. one `ncu --set full` capture of each hot kernel (steady-state launch)
# Outputs land in gpurun_out/prof_<round>/ ; tools/ncu_summary.py turns them
# into profiles/<round>/.
set -e
R=${1:-r01}
MODE=${2:-launches}   # launches | full  (one ncu tool per gpurun call: run the two modes as two calls)
O=gpurun_out/prof_$R
mkdir -p $O
CMD="python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu"
SMALL="python bench.py --envs 512 --steps 1 --warmup 3 --no-e2e --no-cpu"
if [ "$MODE" = launches ]; then
  $CMD > $O/bench_plain.json 2> $O/bench_plain.err
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches.csv $CMD > /dev/null 2>&1
else
  $SMALL > $O/small_plain.json 2>&1
  # one ncu invocation: the first launch of each hot kernel (the third render: the first two are the counters passes, 15 matching launches each, whose raster is raster_kernel<COUNTERS>)
  K='regex:raster_warp_kernel|project_kernel|cull_count_kernel|depth_downsweep|place_downsweep|depth_upsweep|place_upsweep|depth_ties|depth_scan|place_scan'
  ncu --set full --clock-control none --import-source on -k "$K" --launch-skip 30 -c 16 -o $O/full_all $SMALL > $O/ncu_full.log 2>&1 || echo "ncu failed"
fi
ls -la $O
