timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_async.py tests/test_gpu_blur.py -q -x > gpurun_out/pytest_quick.log 2>&1; echo pytest rc=$?; tail -3 gpurun_out/pytest_quick.log
python bench.py > gpurun_out/bench_default.json 2>gpurun_out/bench_default.err; echo bench rc=$?
python -c "
import json; d=json.loads(open('gpurun_out/bench_default.json').read().strip().splitlines()[-1])
print(round(d['value']), 'e2e', round(d['e2e']['value']), 'blocking', round(d['e2e']['value_blocking']), d['config']['chunk_envs'], {k: round(v,2) for k,v in d['roofline']['stage_ms_per_step'].items()}, d['digest'], round(d['roofline']['frac'],3), round(d['roofline']['frac_of_measured'],3))"
bash tools/gpu/quick_launches.sh | grep -E "ties|total"
