mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_residual.py -x -q 2>&1 | tail -15
B="python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:^k_ --csv \
    --log-file gpurun_out/r01_launches.csv $B > gpurun_out/r01_launches.log 2>&1
echo "launches rc=$?"; wc -l gpurun_out/r01_launches.csv
