#!/bin/bash
# Round 2: smoke, full bench (int8 + bf16 learned legs), int8 learned launch list + ncu of the top kernels.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
TAG=${1:-r02a}
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1
echo "smoke rc=$?" >> gpurun_out/${TAG}_smoke.log
timeout 900 python bench.py > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err
echo "bench rc=$?" >> gpurun_out/${TAG}_bench.err
timeout -s KILL 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:^k_ --csv \
   --log-file gpurun_out/${TAG}_i8_launches.csv python scripts/learned_step.py 32 2 i8 > /dev/null 2>&1
echo "launches rc=$?"
for k in k_l8_pair k_l8_attn; do
  timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:$k -s 3 -c 1 \
      -o gpurun_out/${TAG}_$k python scripts/learned_step.py 32 2 i8 > gpurun_out/${TAG}_ncu_$k.log 2>&1
  echo "$k rc=$?"
done
