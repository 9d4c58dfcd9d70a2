mkdir -p gpurun_out
TAG=${1:-r01}
timeout -s KILL 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:^k_ --csv \
   --log-file gpurun_out/${TAG}_learned_launches.csv python scripts/learned_step.py 32 2 > /dev/null 2>&1
echo "launches rc=$?"
for k in k_lt_convpair k_lt_attn_persist; do
  timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:$k -s 2 -c 1 \
      -o gpurun_out/${TAG}_$k python scripts/learned_step.py 32 2 > gpurun_out/${TAG}_ncu_$k.log 2>&1
  echo "$k rc=$?"
done
for k in k_lt_patchify k_upscale9f; do
  timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:$k -s 1 -c 1 \
      -o gpurun_out/${TAG}_$k python scripts/learned_step.py 32 2 > gpurun_out/${TAG}_ncu_$k.log 2>&1
  echo "$k rc=$?"
done
