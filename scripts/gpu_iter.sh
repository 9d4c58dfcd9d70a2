mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
B="python bench.py --steps 20 --warmup 3 --streams 64 --no-cpu-baseline --no-e2e"
timeout 600 $B 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['stages'], d['roofline'])"
for k in k_decode k_packetize k_topk; do
timeout 600 ncu --set full --clock-control none --import-source on -k regex:$k -s 2 -c 1 \
      -o gpurun_out/prof4_$k python bench.py --steps 2 --warmup 1 --streams 16 --no-e2e --no-cpu-baseline > /dev/null 2>&1
echo "ncu $k rc=$?"
done
