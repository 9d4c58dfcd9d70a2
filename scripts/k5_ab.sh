for v in t d; do for b in 16 32; do echo "== $v band $b"; SST_K5_VARIANT=$v SST_K5_BAND=$b timeout -s KILL 200 python scripts/diag/k5_micro.py 2>/dev/null || SST_K5_VARIANT=$v SST_K5_BAND=$b timeout -s KILL 200 python scripts/k5_micro.py; done; done
SST_K5_VARIANT=d timeout -s KILL 300 python -m pytest tests/test_gpu_pipeline.py tests/test_gpu_golden.py -q 2>&1 | tail -1
