# A/B of blocks-per-CTA for cull/project on c3, c4 and one GPU's c5 share
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_async.py -q -x > gpurun_out/pt.log 2>&1; echo pytest rc=$?; tail -2 gpurun_out/pt.log
for L in $LIBS; do
 for v in "" "--config c4" "--config c5 --envs 4096"; do
  GG_LIB=$PWD/$L python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu $v > gpurun_out/ab.json 2>gpurun_out/ab.err; echo "$L $v rc=$?"
  python -c "
import json; d=json.loads(open('gpurun_out/ab.json').read().strip().splitlines()[-1])
print(round(d['value']), {k: round(v,2) for k,v in d['roofline']['stage_ms_per_step'].items()}, d['digest'])"
 done
done
