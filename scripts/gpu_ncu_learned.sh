mkdir -p gpurun_out
TAG=${1:-r01}
timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:k_lt_conv -s 4 -c 1 \
   -o gpurun_out/${TAG}_lt_conv python scripts/bench_learned.py 16 3 > gpurun_out/${TAG}_ncu_lt.log 2>&1
echo "ncu rc=$?"; tail -3 gpurun_out/${TAG}_ncu_lt.log
