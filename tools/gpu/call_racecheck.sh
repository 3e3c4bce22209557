set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
./tools/ubench/alu_peak > gpurun_out/alu_peak.json 2>&1; echo alu rc=$?
cat gpurun_out/alu_peak.json
timeout 900 compute-sanitizer --tool racecheck --racecheck-report hazard python tools/gpu/sanitize_case.py > gpurun_out/racecheck.log 2>&1; echo racecheck rc=$?
tail -30 gpurun_out/racecheck.log
