for c in 1024 4096 0; do
python bench.py --chunk $c --no-cpu > gpurun_out/ab.json 2>gpurun_out/ab.err; echo "chunk $c rc=$?"
python -c "
import json; d=json.loads(open('gpurun_out/ab.json').read().strip().splitlines()[-1])
print(round(d['value']), 'e2e', round(d['e2e']['value']), 'blocking', round(d['e2e']['value_blocking']))"
done
nvidia-smi --query-gpu=memory.used,memory.total --format=csv
