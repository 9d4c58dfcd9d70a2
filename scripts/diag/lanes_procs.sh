# A/B: lanes per process and processes per GPU (SST_BENCH_SHARE_GPU hook)
B="--steps 20 --warmup 3 --no-e2e --no-cpu-baseline --no-learned --no-rgb24"
for l in 2 4 8; do
  timeout -s KILL 400 python bench.py $B --lanes $l > gpurun_out/la.json 2>/dev/null
  python -c "import json; d=json.loads(open('gpurun_out/la.json').read().strip().splitlines()[-1]); print('1 proc, lanes $l', d['value'], d['ms_per_step'])"
done
for l in 2 4; do
  SST_BENCH_SHARE_GPU=1 timeout -s KILL 600 python bench.py $B --gpus 2 --lanes $l > gpurun_out/la.json 2>/dev/null
  python -c "import json; d=json.loads(open('gpurun_out/la.json').read().strip().splitlines()[-1]); print('2 procs, lanes $l', d['value'], [r['ms'] for r in d['per_rank']])"
done
timeout -s KILL 400 python bench.py $B --streams 128 > gpurun_out/la.json 2>/dev/null
python -c "import json; d=json.loads(open('gpurun_out/la.json').read().strip().splitlines()[-1]); print('1 proc, 128 streams', d['value'], d['ms_per_step'])"
