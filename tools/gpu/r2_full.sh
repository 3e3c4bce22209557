# full GPU suite + default bench line
bash tools/gpu/r2_tests.sh
python bench.py > gpurun_out/bench_default.json 2>gpurun_out/bench_default.err; echo bench rc=$?
python -c "
import json; d=json.loads(open('gpurun_out/bench_default.json').read().strip().splitlines()[-1])
print(round(d['value']), 'e2e', round(d['e2e']['value']), 'blocking', round(d['e2e']['value_blocking']), d['config']['chunk_envs'], {k: round(v,2) for k,v in d['roofline']['stage_ms_per_step'].items()}, d['digest'], round(d['roofline']['frac'],3), round(d['roofline']['frac_of_measured'],3))"
