# project storage blocks per CTA (GG_PROJ_BPC, a temporary switch; measured 1: 25.30, 2: 25.55, 4: 25.43 ms) A/B, then the parity subsets that cover the cull/project paths
for B in 0 2 4 0 2 4; do
  GG_PROJ_BPC=$B python bench.py --no-e2e --no-cpu > gpurun_out/ab.json 2>gpurun_out/ab.err; echo "proj bpc=$B rc=$?"
  python -c "
import json; d=json.loads(open('gpurun_out/ab.json').read().strip().splitlines()[-1])
print(round(d['value']), {k: round(v,2) for k,v in d['roofline']['stage_ms_per_step'].items()}, d['digest'])"
done
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_async.py -x -q -m gpu 2>&1 | tail -5
