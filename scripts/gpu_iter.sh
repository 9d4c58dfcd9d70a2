mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
timeout 600 python bench.py --no-cpu-baseline --no-e2e 2>&1 | tail -1 > gpurun_out/bench_iter.json
python -c "import json; d=json.load(open('gpurun_out/bench_iter.json')); print(d['value'], d['stages'], d['roofline']['frac'], d['path_roofline']['frac'], d['gpu_launches'])"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_upscale_blend_tma -s 2 -c 1 \
      -o gpurun_out/prof5_k5 python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > /dev/null 2>&1; echo "ncu rc=$?"
