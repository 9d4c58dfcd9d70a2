cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_learned.py -x -q -p no:cacheprovider 2>&1 | tail -3
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/r02d_bench.json 2> gpurun_out/r02d_bench.err
echo "bench rc=$?"; tail -3 gpurun_out/r02d_bench.err
