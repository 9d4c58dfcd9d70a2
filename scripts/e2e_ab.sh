free -g | head -2
for e in 8 16; do timeout -s KILL 500 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-learned --e2e-streams $e > gpurun_out/e2e.json 2>gpurun_out/e2e.err; python -c "import json; d=json.load(open('gpurun_out/e2e.json')); print('E=$e', d['e2e']['value'], d['e2e']['wall_s'])"; done
