# K5 A/B: direct streaming stores (default) vs TMA-store tiles, with TMA or
# register-staged window loads; then parity with each store variant
for v in direct tiles; do for l in tma sync; do echo "== $v / $l"; SST_K5_VARIANT=$v SST_K5_LOAD=$l timeout -s KILL 200 python scripts/k5_micro.py; done; done
for v in direct tiles; do SST_K5_VARIANT=$v timeout -s KILL 600 python -m pytest tests/test_gpu_pipeline.py tests/test_gpu_golden.py tests/test_gpu_api.py -q 2>&1 | tail -1; done
