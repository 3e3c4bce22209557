timeout 900 python -m pytest tests/test_gpu_blur.py tests/test_gpu_parity.py -q -x > gpurun_out/pytest_blur.log 2>&1; echo pytest rc=$?; tail -3 gpurun_out/pytest_blur.log
for K in 3 4; do
python bench.py --blur $K --no-e2e --no-cpu > gpurun_out/blur$K.json 2>gpurun_out/blur$K.err; echo "blur $K rc=$?"
python -c "
import json; d=json.loads(open('gpurun_out/blur$K.json').read().strip().splitlines()[-1])
print(round(d['value']), round(d['ms_per_step'],1), {k: round(v,2) for k,v in d['roofline']['stage_ms_per_step'].items()})"
done
