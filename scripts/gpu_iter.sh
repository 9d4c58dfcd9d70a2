mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
timeout 600 python bench.py --no-cpu-baseline 2>&1 | tail -1 > gpurun_out/bench_iter.json
python -c "import json; d=json.load(open('gpurun_out/bench_iter.json')); print(d['value'], d['stages'], d['roofline'], d['path_roofline'], d['e2e']['value'])"
