# GG_ASYNC_LOOP A/B: async/graph mode with bounded-grid LOOP kernels (1) or capacity-sized grids of the sync kernels (0)
for V in 1 0 1 0; do
  GG_ASYNC_LOOP=$V python bench.py --mode graph --no-e2e --no-cpu > gpurun_out/ab.json 2>gpurun_out/ab.err; echo "loop=$V rc=$?"
  python -c "
import json; d=json.loads(open('gpurun_out/ab.json').read().strip().splitlines()[-1])
print(round(d['value']), {k: round(v,2) for k,v in d['roofline']['stage_ms_per_step'].items()}, d['digest'])"
done
GG_ASYNC_LOOP=0 timeout 900 python -m pytest tests/test_gpu_async.py tests/test_gpu_rate_decoupled.py -x -q -m gpu 2>&1 | tail -2
