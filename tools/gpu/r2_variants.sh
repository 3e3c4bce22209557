# round-2 evidence: the default bench line (with e2e and the CPU oracle), then
# SURVEY §8(d).3 separate runs and the other configs, one JSON line each
mkdir -p gpurun_out/var2
python bench.py > gpurun_out/var2/default.json 2> gpurun_out/var2/default.err; echo default rc=$?
B="python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu"
i=0
for v in "--outputs rgb" "--outputs depth" "--sh 0" "--tiles paper" "--tiles ellipse" "--mode async" "--mode graph" "--config c4 --scenes 128" "--config c4" "--config c2" "--config c1" "--blur 3" "--config c5 --envs 4096" "--config c1 --mode graph"; do
  i=$((i+1))
  $B $v > gpurun_out/var2/v$i.json 2>gpurun_out/var2/v$i.err; echo "$v rc=$?"
  python -c "
import json;d=json.loads(open('gpurun_out/var2/v$i.json').read().strip().splitlines()[-1])
print('$v'.ljust(24), round(d['value']), round(d['ms_per_step'],1), {k: round(v,1) for k,v in d['roofline']['stage_ms_per_step'].items()}, 'raster frac', round(d['roofline_path']['kernels']['raster']['frac'],3), d['digest'], d.get('load_s'))" || tail -3 gpurun_out/var2/v$i.err
done
