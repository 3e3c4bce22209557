# SURVEY §8(d).3 separate runs: RGB+D (headline), RGB-only, depth-only, d=0, paper tile rects, async mode
B="python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu"
for v in "" "--outputs rgb" "--outputs depth" "--sh 0" "--tiles paper" "--mode async" "--config c4 --scenes 128"; do
  $B $v > gpurun_out/var.json 2>gpurun_out/var.err
  python -c "
import json;d=json.load(open('gpurun_out/var.json'))
rp=d['roofline_path']
print('$v'.ljust(16), round(d['value']), 'path_frac', round(rp['frac'],3), {k:(round(v['alg_ms'],1),round(v['measured_ms'],1),v['bound']) for k,v in rp['stages'].items()})" || tail -3 gpurun_out/var.err
done
