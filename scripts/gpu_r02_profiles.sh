#!/bin/bash
# Round-2 evidence run: full GPU test suite, the default bench, ncu launch
# lists + --set full captures (main path and the int8 learned path), and
# compute-sanitizer over the new int8 kernels.  Outputs under gpurun_out/.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
TAG=${1:-r02}
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/${TAG}_gputest.log 2>&1
echo "pytest rc=$?" | tee -a gpurun_out/${TAG}_gputest.log
tail -2 gpurun_out/${TAG}_gputest.log
timeout 900 python bench.py > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err
echo "bench rc=$?"
# main path (the bench workload, 64 x 1080p streams)
B="python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --no-learned"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:^k_ --csv \
    --log-file gpurun_out/${TAG}_launches.csv $B > gpurun_out/${TAG}_launches.log 2>&1
echo "launches rc=$?"
for k in k_upscale_blend_tma k_encode k_decode k_packetize k_topk k_parse; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$k -s 2 -c 1 \
      -o gpurun_out/${TAG}_$k $B > gpurun_out/${TAG}_ncu_$k.log 2>&1
  echo "$k rc=$?"
done
# int8 learned path (32 x 1080p GoPs per step)
timeout -s KILL 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:^k_ --csv \
   --log-file gpurun_out/${TAG}_learned_launches.csv python scripts/learned_step.py 32 2 i8 > /dev/null 2>&1
echo "learned launches rc=$?"
for spec in "k_l8_pair:3" "k_l8_attn:1" "k_l8_patchify:1" "k_upscale9f:1"; do
  k=${spec%%:*}; sk=${spec##*:}
  timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:$k -s $sk -c 1 \
      -o gpurun_out/${TAG}_$k python scripts/learned_step.py 32 2 i8 > gpurun_out/${TAG}_ncu_$k.log 2>&1
  echo "$k rc=$?"
done
CS=/usr/local/cuda/bin/compute-sanitizer
timeout -s KILL 900 $CS --tool memcheck --error-exitcode 9 --print-limit 20 python -m pytest tests/test_gpu_learned_i8.py -q -x -k "not 1080 and not 720 and not gop_codec" > gpurun_out/${TAG}_san_i8.log 2>&1; echo "memcheck i8 rc=$?"
timeout -s KILL 900 $CS --tool racecheck --error-exitcode 9 --print-limit 20 python -m pytest tests/test_gpu_learned_i8.py -q -x -k "attention_core and 13" > gpurun_out/${TAG}_san_race_i8.log 2>&1; echo "racecheck i8 attn rc=$?"
timeout -s KILL 900 $CS --tool memcheck --error-exitcode 9 --print-limit 20 python -m pytest tests/test_gpu_residual.py tests/test_gpu_metrics.py -q -x -k "not 1080" > gpurun_out/${TAG}_san_rc.log 2>&1; echo "memcheck rc/metrics rc=$?"
timeout -s KILL 900 $CS --tool racecheck --error-exitcode 9 --print-limit 20 python -m pytest tests/test_gpu_residual.py -q -x -k "batched_coding" > gpurun_out/${TAG}_san_race_rc.log 2>&1; echo "racecheck rc encoder rc=$?"
timeout -s KILL 900 $CS --tool racecheck --error-exitcode 9 --print-limit 20 python -m pytest tests/test_gpu_learned_i8.py -q -x -k "patchify_haar and 128" > gpurun_out/${TAG}_san_race_haar.log 2>&1; echo "racecheck haar rc=$?"
ls gpurun_out | grep "^${TAG}" | head -50
