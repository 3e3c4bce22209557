timeout 1200 python -m pytest tests/test_gpu_dist.py tests/test_gpu_fullsize.py -q -x -k "dist or c3_sampled_bench" > gpurun_out/pytest_dist.log 2>&1; echo pytest rc=$?; tail -15 gpurun_out/pytest_dist.log
python bench.py > gpurun_out/bench_default.json 2>gpurun_out/bench_default.err; echo bench rc=$?
python -c "
import json; d=json.loads(open('gpurun_out/bench_default.json').read().strip().splitlines()[-1])
print(round(d['value']), d['e2e']['value'], {k: round(v,2) for k,v in d['roofline']['stage_ms_per_step'].items()}, d['digest'], d['load_s'], d['roofline']['frac'])"
