mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_pipeline.py tests/test_gpu_golden.py -x -q 2>&1 | tail -2
for cfg in "32 1" "32 2" "16 1" "16 2"; do
set -- $cfg
SST_K5_BAND=$1 SST_K5_NBUF=$2 timeout 600 python bench.py --no-cpu-baseline --no-e2e 2>&1 | tail -1 > gpurun_out/bench_ab.json
python -c "import json; d=json.load(open('gpurun_out/bench_ab.json')); print('band $1 nbuf $2', d['value'], d['stages']['K5_upscale_blend'], d['roofline']['frac'], d['path_roofline']['frac'])"
done
