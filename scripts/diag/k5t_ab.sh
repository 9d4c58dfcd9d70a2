for sm in 0 30000 45000; do SST_K5T_SMEM=$sm SST_BENCH_FUSED=1 timeout 300 python bench.py --steps 20 --no-e2e --no-cpu-baseline --no-learned --no-rgb24 > gpurun_out/ab.json 2>gpurun_out/ab.err; python -c "
import json;d=json.loads(open('gpurun_out/ab.json').read().strip().splitlines()[-1])
print('smem $sm', d['value'],d['ms_per_step'],d['stages']['K5_upscale_blend']['ms_per_launch'])"; done
