# GPU tests with durations (no -x: report every failure)
nproc
timeout 2400 python -m pytest tests -m gpu -q --durations=20 > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?
grep -E "passed|failed|Tally|Error|FAILED" gpurun_out/pytest_gpu.log | tail -40
tail -25 gpurun_out/pytest_gpu.log
