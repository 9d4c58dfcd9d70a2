#!/bin/bash
# Late round-2 evidence run: full GPU tests, smoke, the default bench, ncu
# launch list of the bench workload, --set full captures of the main-path
# kernels (K5 v2, K1), the raw-rgb24 kernels and K5-9, and compute-sanitizer
# over the raw-rgb24 / blend-edge tests.  Outputs under gpurun_out/.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
TAG=${1:-r02s3}
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/${TAG}_gputest.log 2>&1
echo "pytest rc=$?"; tail -2 gpurun_out/${TAG}_gputest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1; echo "smoke rc=$?"
timeout 1200 python bench.py > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err; echo "bench rc=$?"
B="python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --no-learned --no-rgb24"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:^k_ --csv \
    --log-file gpurun_out/${TAG}_launches.csv $B > /dev/null 2>&1; echo "launches rc=$?"
for k in k_upscale_blend_v2 k_encode; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$k -s 2 -c 1 \
      -o gpurun_out/${TAG}_$k $B > /dev/null 2>&1; echo "$k rc=$?"
done
for k in k_encode_u8 k_upscale_blend_u8f; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$k -s 1 -c 1 \
      -o gpurun_out/${TAG}_$k python scripts/rgb24_prof.py 3 > /dev/null 2>&1; echo "$k rc=$?"
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:^k_ --csv \
    --log-file gpurun_out/${TAG}_rgb24_launches.csv python bench.py --steps 2 --warmup 1 --no-e2e \
    --no-cpu-baseline --no-learned > /dev/null 2>&1; echo "rgb24 launches rc=$?"
CS=/usr/local/cuda/bin/compute-sanitizer
timeout -s KILL 900 $CS --tool memcheck --error-exitcode 9 --print-limit 20 python -m pytest tests/test_gpu_rgb24.py tests/test_gpu_blend_edge.py -q -x -k "not 1080" > gpurun_out/${TAG}_san_mem.log 2>&1; echo "memcheck rc=$?"
timeout -s KILL 900 $CS --tool racecheck --error-exitcode 9 --print-limit 20 python -m pytest tests/test_gpu_rgb24.py -q -x -k "encode_u8_equals and 48" > gpurun_out/${TAG}_san_race.log 2>&1; echo "racecheck k1u8 rc=$?"
timeout -s KILL 900 $CS --tool synccheck --error-exitcode 9 --print-limit 20 python -m pytest tests/test_gpu_rgb24.py -q -x -k "encode_u8_equals and 48" > gpurun_out/${TAG}_san_sync.log 2>&1; echo "synccheck k1u8 rc=$?"
ls gpurun_out | grep "^${TAG}" | head -40
