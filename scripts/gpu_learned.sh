mkdir -p gpurun_out
timeout -s KILL 400 python -m pytest tests/test_gpu_learned.py -x -q > gpurun_out/learned.log 2>&1; echo "learned rc=$?"
tail -40 gpurun_out/learned.log
