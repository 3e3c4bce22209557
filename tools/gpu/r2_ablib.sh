# A/B of in-tree library builds: bench (c3, no e2e/cpu) per GG_LIB in $LIBS
for L in $LIBS; do
  GG_LIB=$PWD/$L python bench.py --no-e2e --no-cpu > gpurun_out/ab.json 2>gpurun_out/ab.err; echo "$L rc=$?"
  python -c "
import json; d=json.loads(open('gpurun_out/ab.json').read().strip().splitlines()[-1])
print(round(d['value']), {k: round(v,2) for k,v in d['roofline']['stage_ms_per_step'].items()}, d['digest'])"
done
