# A/B of env-selected kernel variants: -m gpu tests (default), parity tests
# under each variant, then the default bench once per variant setting.
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?; tail -2 gpurun_out/pytest_gpu.log
for v in ${VARIANTS:-"X=1"}; do
  env $v timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_depth_only.py -m gpu -q -x > gpurun_out/pytest_v.log 2>&1; echo "$v parity rc=$?"; tail -1 gpurun_out/pytest_v.log
done
B="python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu"
for v in ${VARIANTS:-"X=1"}; do
  env $v $B > gpurun_out/ab.json 2>gpurun_out/ab.err
  python -c "import json;d=json.load(open('gpurun_out/ab.json'));print('$v', round(d['value']), {k:round(x,2) for k,x in d['roofline']['stage_ms_per_step'].items()}, d['digest'])" || tail -3 gpurun_out/ab.err
done
