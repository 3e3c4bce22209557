# quick parity + bench + launch list + ncu --set full of kernels matching $K (512-env run)
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_tight.py tests/test_gpu_async.py -q -x > gpurun_out/pytest_quick.log 2>&1; echo pytest rc=$?; tail -2 gpurun_out/pytest_quick.log
python bench.py --no-e2e --no-cpu > gpurun_out/ab.json 2>gpurun_out/ab.err; echo "bench rc=$?"
python -c "
import json; d=json.loads(open('gpurun_out/ab.json').read().strip().splitlines()[-1])
print(round(d['value']), {k: round(v,2) for k,v in d['roofline']['stage_ms_per_step'].items()}, d['digest'])"
bash tools/gpu/quick_launches.sh
SMALL="python bench.py --envs 512 --steps 1 --warmup 3 --no-e2e --no-cpu"
$SMALL > gpurun_out/small_plain.json 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"${K:-depth_ties|place_downsweep}" -s 2 -c 2 -o gpurun_out/prof_r2 $SMALL > gpurun_out/ncu_prof.log 2>&1; tail -2 gpurun_out/ncu_prof.log
