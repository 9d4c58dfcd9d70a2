mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
for L in 2 4; do
timeout 600 python bench.py --no-cpu-baseline --no-e2e --lanes $L 2>&1 | tail -1 > gpurun_out/bench_iter.json
python -c "import json; d=json.load(open('gpurun_out/bench_iter.json')); print('lanes $L', d['value'], d['stages'], d['roofline']['frac'], d['path_roofline']['frac'], d['gpu_launches'])"
done
