# cull storage blocks per CTA (GG_CULL_BPC) per library build: "lib:bpc" pairs in $RUNS
for RB in $RUNS; do
  L=${RB%%:*}; B=${RB##*:}
  GG_LIB=$PWD/$L GG_CULL_BPC=$B python bench.py --no-e2e --no-cpu > gpurun_out/ab.json 2>gpurun_out/ab.err; echo "$L bpc=$B rc=$?"
  python -c "
import json; d=json.loads(open('gpurun_out/ab.json').read().strip().splitlines()[-1])
print(round(d['value']), {k: round(v,2) for k,v in d['roofline']['stage_ms_per_step'].items()}, d['digest'])"
done
