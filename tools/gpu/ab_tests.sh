# tests and bench under each VARIANTS env setting (e.g. VARIANTS="GG_RASTER=w GG_RASTER=h")
for v in ${VARIANTS:-"X=1"}; do
  env $v timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "$v pytest: $(tail -1 gpurun_out/pytest_gpu.log)"
  env $v python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu > gpurun_out/ab.json 2>gpurun_out/ab.err
  python -c "import json;d=json.load(open('gpurun_out/ab.json'));print('$v', round(d['value']), d['roofline']['stage_ms_per_step'], d['digest'])" || tail -3 gpurun_out/ab.err
done
