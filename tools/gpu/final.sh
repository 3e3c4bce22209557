set -x
mkdir -p gpurun_out/fin
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/fin/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/fin/smoke.log
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/fin/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/fin/pytest_gpu.log
python bench.py > gpurun_out/fin/bench_default.json 2> gpurun_out/fin/bench_default.err
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/fin/launches.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu > /dev/null 2>&1
echo done
