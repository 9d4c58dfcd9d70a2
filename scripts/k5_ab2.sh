echo "== micro band16 nbuf1"; SST_K5_BAND=16 SST_K5_NBUF=1 timeout -s KILL 200 python scripts/k5_micro.py
for cfg in "32 2" "16 1" "32 1"; do set -- $cfg
SST_K5_BAND=$1 SST_K5_NBUF=$2 timeout -s KILL 400 python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu-baseline --no-learned > gpurun_out/ab.json 2>/dev/null
python -c "import json; d=json.load(open('gpurun_out/ab.json')); print('band $1 nbuf $2', d['value'], d['stages']['K5_upscale_blend'], d['roofline']['frac'])"
done
