#!/bin/bash
# Round-2 GPU check: full -m gpu suite, default bench, 2-rank shared-GPU bench.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
nproc > gpurun_out/r02_host.txt; free -g >> gpurun_out/r02_host.txt; nvidia-smi -L >> gpurun_out/r02_host.txt
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider ${PYTEST_ARGS} > gpurun_out/r02_gputest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r02_gputest.log
timeout 600 python bench.py > gpurun_out/r02_bench.json 2> gpurun_out/r02_bench.err
echo "bench rc=$?" >> gpurun_out/r02_bench.err
SST_BENCH_SHARE_GPU=1 timeout 600 python bench.py --gpus 2 --no-learned --steps 10 --warmup 3 > gpurun_out/r02_bench2.json 2> gpurun_out/r02_bench2.err
echo "bench2 rc=$?" >> gpurun_out/r02_bench2.err
tail -3 gpurun_out/r02_gputest.log
