# e2e (host-buffer path) A/B: default bench without the CPU leg, once per VARIANTS setting
for v in ${VARIANTS:-"X=1"}; do
  env $v python bench.py --no-cpu > gpurun_out/e2e_ab.json 2> gpurun_out/e2e_ab.err
  python -c "import json;d=[json.loads(l) for l in open('gpurun_out/e2e_ab.json') if l.startswith('{')][-1];print('$v', round(d['value']), round(d['e2e']['value']), d['digest'])" || tail -3 gpurun_out/e2e_ab.err
done
