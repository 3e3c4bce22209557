# quick: gpu tests + 512-env launch list (kernel times)
timeout 600 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?; tail -3 gpurun_out/pytest_gpu.log
CMD="python bench.py --envs 512 --steps 1 --warmup 1 --no-e2e --no-cpu --mode ${MODE:-sync}"
$CMD > gpurun_out/b512.json 2> gpurun_out/b512.err && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_q.csv $CMD > /dev/null 2>&1
python - <<'PY'
import csv, collections
rows=list(csv.reader(open('gpurun_out/launches_q.csv')))
hdr=[i for i,r in enumerate(rows) if 'Kernel Name' in r][0]
h=rows[hdr]; ki=h.index('Kernel Name'); vi=h.index('Metric Value')
rs=rows[hdr+1:]
# last render = the final N launches after the last setup_envs
last=max(i for i,r in enumerate(rs) if 'setup_envs' in r[ki])
agg=collections.OrderedDict()
for r in rs[last:]:
    k=r[ki].split('(')[0].replace('void ','')[:40]
    agg[k]=agg.get(k,0)+float(r[vi])
for k,v in agg.items(): print(f"{k:42s} {v/1e6:8.3f} ms")
print('total', sum(agg.values())/1e6)
PY
