# blur bench per library build in $LIBS (GG_LIB), --blur 3
for L in $LIBS; do
  GG_LIB=$PWD/$L python bench.py --blur 3 --steps 3 --warmup 3 --no-e2e --no-cpu > gpurun_out/ab.json 2>gpurun_out/ab.err; echo "$L rc=$?"
  python -c "
import json; d=json.loads(open('gpurun_out/ab.json').read().strip().splitlines()[-1])
print(round(d['value']), {k: round(v,2) for k,v in d['roofline']['stage_ms_per_step'].items()}, d['digest'])"
done
