# ncu evidence for profiles/ at the bench's own workload (64 x 1080p streams).
#   1. launch list of `bench.py` (our kernels only), 2 timed steps
#   2. --set full capture of one launch of each pipeline kernel
mkdir -p gpurun_out
TAG=${1:-r01}
B="python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --no-learned"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:^k_ --csv \
    --log-file gpurun_out/${TAG}_launches.csv $B > gpurun_out/${TAG}_launches.log 2>&1
echo "launches rc=$?"
for k in k_upscale_blend_tma k_encode k_decode k_packetize k_topk k_parse; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$k -s 2 -c 1 \
      -o gpurun_out/${TAG}_$k $B > gpurun_out/${TAG}_ncu_$k.log 2>&1
  echo "$k rc=$?"
done
ls -la gpurun_out | grep $TAG
