# per-kernel ms of one 1024-env render (ncu launch list), once per VARIANTS env setting
CMD="python bench.py --envs 1024 --steps 1 --warmup 3 --no-e2e --no-cpu --mode ${MODE:-sync} ${EXTRA}"
for v in ${VARIANTS:-"X=1"}; do
  echo "== $v"
  env $v $CMD > gpurun_out/b1024.json 2> gpurun_out/b1024.err && \
  env $v ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_q.csv $CMD > /dev/null 2>&1
  python - <<'PY'
import csv, collections
rows=list(csv.reader(open('gpurun_out/launches_q.csv')))
hdr=[i for i,r in enumerate(rows) if 'Kernel Name' in r][0]
h=rows[hdr]; ki=h.index('Kernel Name'); vi=h.index('Metric Value')
rs=rows[hdr+1:]
last=max(i for i,r in enumerate(rs) if 'setup_envs' in r[ki])
agg=collections.OrderedDict()
for r in rs[last:]:
    k=r[ki].split('(')[0].replace('void ','')[:40]
    agg[k]=agg.get(k,0)+float(r[vi])
for k,v in agg.items(): print(f"{k:42s} {v/1e6:8.3f} ms")
print('total', sum(agg.values())/1e6)
PY
done
