cd $GRAFT_REPO_ROOT
echo "== f64 windows (default)"; python scripts/k5_9_micro.py
echo "== f32 windows"; SST_K5_9W=f32 python scripts/k5_9_micro.py
timeout 600 python -m pytest tests/test_gpu_upscale9.py tests/test_gpu_learned_i8.py -x -q -p no:cacheprovider 2>&1 | tail -3
