# variants.sh plus c2, graph mode and one GPU's share of c5, all at one commit
bash tools/gpu/variants.sh > gpurun_out/variants.txt 2>&1
B="python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu"
for v in "--mode graph" "--config c2"; do
  $B $v > gpurun_out/var.json 2>gpurun_out/var.err
  python -c "import json;d=json.load(open('gpurun_out/var.json'));print('$v'.ljust(16), round(d['value']), 'path_frac', round(d['roofline_path']['frac'],3))" >> gpurun_out/variants.txt || tail -3 gpurun_out/var.err >> gpurun_out/variants.txt
done
timeout 1200 python bench.py --config c5 --envs 4096 --steps 5 --warmup 3 --no-e2e --no-cpu > gpurun_out/bench_c5_per_gpu.json 2> gpurun_out/c5.err
echo "c5 rc=$?" >> gpurun_out/variants.txt
