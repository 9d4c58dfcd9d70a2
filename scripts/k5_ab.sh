# K5 A/B: register-staged vs TMA I/P window loads, then parity with each
for v in sync tma; do echo "== $v"; SST_K5_LOAD=$v timeout -s KILL 200 python scripts/k5_micro.py; done
for v in sync tma; do SST_K5_LOAD=$v timeout -s KILL 600 python -m pytest tests/test_gpu_pipeline.py tests/test_gpu_golden.py -q 2>&1 | tail -1; done
