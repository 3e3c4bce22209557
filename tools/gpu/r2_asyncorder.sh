# device-side env order for the sync-free path: graph-mode bench per library build in $LIBS (c3 and c4 128 scenes)
for L in $LIBS; do
  for C in "" "--config c4 --scenes 128"; do
    GG_LIB=$PWD/$L python bench.py $C --mode graph --steps 5 --warmup 3 --no-e2e --no-cpu > gpurun_out/ab.json 2>gpurun_out/ab.err; echo "$L $C rc=$?"
    python -c "
import json; d=json.loads(open('gpurun_out/ab.json').read().strip().splitlines()[-1])
print(round(d['value']), {k: round(v,2) for k,v in d['roofline']['stage_ms_per_step'].items()}, d['digest'])"
  done
done
