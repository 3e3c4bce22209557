for c in 1024 2048 4096; do
  python bench.py --no-e2e --no-cpu --chunk $c > gpurun_out/ab.json 2>gpurun_out/ab.err; echo "chunk $c rc=$?"
  python -c "
import json; d=json.loads(open('gpurun_out/ab.json').read().strip().splitlines()[-1])
print(round(d['value']), {k: round(v,2) for k,v in d['roofline']['stage_ms_per_step'].items()}, d['digest'])"
done
CMD="python bench.py --config c1 --steps 3 --warmup 3 --no-e2e --no-cpu"
$CMD > gpurun_out/c1.json 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c1.csv $CMD > /dev/null 2>&1
python - <<'PY'
import csv
rows=list(csv.reader(open('gpurun_out/launches_c1.csv')))
hdr=[i for i,r in enumerate(rows) if 'Kernel Name' in r][0]
h=rows[hdr]; ki=h.index('Kernel Name'); vi=h.index('Metric Value')
rs=rows[hdr+1:]
last=max(i for i,r in enumerate(rs) if 'setup_envs' in r[ki])
tot=0
for r in rs[last:]:
    print(r[ki].split('(')[0][:50], float(r[vi])/1e3, 'us'); tot+=float(r[vi])
print('total us', tot/1e3, 'launches', len(rs)-last)
PY
