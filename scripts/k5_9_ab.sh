for v in "32,1" "f9,16" "f9,32"; do echo "== $v"; SST_K5_9=$v timeout -s KILL 200 python scripts/k5_9_micro.py; done
for v in "f9,16" "f9,32"; do SST_K5_9=$v timeout -s KILL 300 python -m pytest tests/test_gpu_learned.py -q -k gop_codec 2>&1 | tail -1; done
