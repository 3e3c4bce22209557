# quick parity subset + 1024-env launch list + default bench value
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_tight.py tests/test_gpu_async.py -q -x > gpurun_out/pytest_quick.log 2>&1; echo pytest rc=$?; tail -2 gpurun_out/pytest_quick.log
python bench.py --no-e2e --no-cpu > gpurun_out/ab.json 2>gpurun_out/ab.err; echo "bench rc=$?"
python -c "
import json; d=json.loads(open('gpurun_out/ab.json').read().strip().splitlines()[-1])
print(round(d['value']), {k: round(v,2) for k,v in d['roofline']['stage_ms_per_step'].items()}, d['digest'])"
bash tools/gpu/quick_launches.sh
