# round-2 check: GPU tests (with durations), then the default bench
set -x
nproc
timeout 1500 python -m pytest tests -m gpu -q -x --durations=15 > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?
tail -30 gpurun_out/pytest_gpu.log
timeout 600 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; echo bench rc=$?
tail -c 3000 gpurun_out/bench_default.json; tail -5 gpurun_out/bench_default.err
