for l in 1 2 4; do timeout -s KILL 400 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --learned-lanes $l > gpurun_out/ll.json 2>gpurun_out/ll.err; python -c "import json; d=json.load(open('gpurun_out/ll.json'))['learned_tokenizer']; print('lanes $l', d['value'], d['ms_per_step'], d['roofline']['frac'])"; done
tail -3 gpurun_out/ll.err
