mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
B="python bench.py --steps 20 --warmup 3 --streams 64 --no-cpu-baseline --no-e2e"
SST_K5_VARIANT=2 timeout 600 $B 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('v2', d['value'], d['stages'], d['roofline']['frac'])"
timeout 600 $B 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('v3d', d['value'], d['stages'], d['roofline']['frac'])"
for k in k_upscale_blend_tma k_decode; do
timeout 600 ncu --set full --clock-control none --import-source on -k regex:$k -s 2 -c 1 \
      -o gpurun_out/prof2_$k python bench.py --steps 2 --warmup 1 --streams 16 --no-e2e --no-cpu-baseline > /dev/null 2>&1
echo "ncu $k rc=$?"
done
