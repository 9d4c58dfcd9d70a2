# ncu evidence for profiles/: launch list of one bench step + full captures of the top kernels
mkdir -p gpurun_out
B="python bench.py --steps 2 --warmup 1 --streams 16 --no-e2e --no-cpu-baseline"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launches.csv $B > gpurun_out/ncu_launches.log 2>&1
echo "launches rc=$?"
for k in k_upscale_blend k_encode k_decode k_packetize k_topk k_parse; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$k -s 2 -c 1 \
      -o gpurun_out/prof_$k $B > gpurun_out/ncu_$k.log 2>&1
  echo "$k rc=$?"
done
ls -la gpurun_out
