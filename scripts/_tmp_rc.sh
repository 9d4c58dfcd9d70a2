cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_gpu_residual.py tests/test_gpu_streamfile.py -x -q -p no:cacheprovider 2>&1 | tail -3
echo "== cum (default)"; python scripts/bench_residual.py 32
