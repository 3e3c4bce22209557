timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "render_host" > gpurun_out/pytest_host.log 2>&1; echo pytest rc=$?; tail -2 gpurun_out/pytest_host.log
python bench.py > gpurun_out/bench_default.json 2>gpurun_out/bench_default.err; echo bench rc=$?
python -c "
import json; d=json.loads(open('gpurun_out/bench_default.json').read().strip().splitlines()[-1])
print(round(d['value']), 'e2e', round(d['e2e']['value']), 'blocking', round(d['e2e']['value_blocking']), {k: round(v,2) for k,v in d['roofline']['stage_ms_per_step'].items()}, d['digest'], d['roofline']['frac'], d['cpu_baseline'])"
tail -3 gpurun_out/bench_default.err
free -g | head -2
