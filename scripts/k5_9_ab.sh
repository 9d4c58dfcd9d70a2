# K5-9 A/B: register-staged vs cp.async vs TMA window loads, then parity
for v in sync async tma; do echo "== $v"; SST_K5_9=$v timeout -s KILL 200 python scripts/k5_9_micro.py; done
for v in sync async tma; do SST_K5_9=$v timeout -s KILL 300 python -m pytest tests/test_gpu_learned.py -q -k "gop_codec or upscale" 2>&1 | tail -1; done
