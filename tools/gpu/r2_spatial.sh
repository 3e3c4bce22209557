timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_tight.py tests/test_gpu_async.py tests/test_gpu_blur.py tests/test_gpu_depth_only.py -q -x > gpurun_out/pytest_quick.log 2>&1; echo pytest rc=$?; tail -5 gpurun_out/pytest_quick.log
timeout 900 python -m pytest tests/test_gpu_fullsize.py -q -x -k "c3_sampled_bench or c4" > gpurun_out/pytest_full.log 2>&1; echo full rc=$?; tail -5 gpurun_out/pytest_full.log
python bench.py --no-e2e --no-cpu > gpurun_out/b_spatial.json 2>gpurun_out/b_spatial.err; echo bench rc=$?
GG_NO_SPATIAL_ORDER=1 python bench.py --no-e2e --no-cpu > gpurun_out/b_input.json 2>gpurun_out/b_input.err; echo bench2 rc=$?
python - <<'PY'
import json
for f in ("gpurun_out/b_spatial.json","gpurun_out/b_input.json"):
    try:
        d=json.loads(open(f).read().strip().splitlines()[-1])
        print(f, round(d["value"]), {k: round(v,2) for k,v in d["roofline"]["stage_ms_per_step"].items()}, d["digest"])
    except Exception as e:
        print(f, "ERR", e, open(f.replace('.json','.err')).read()[-2000:])
PY
