#!/bin/bash
# Closing evidence run of round 2: full GPU tests, smoke, the default bench
# and a --set full capture of the raw-rgb24 K5 (32-row bands).
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
TAG=${1:-r02s10}
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/${TAG}_gputest.log 2>&1
echo "pytest rc=$?"; tail -2 gpurun_out/${TAG}_gputest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1; echo "smoke rc=$?"
timeout 1200 python bench.py > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err; echo "bench rc=$?"
timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:k_upscale_blend_u8f -s 1 -c 1 \
    -f -o gpurun_out/${TAG}_k5u8f python scripts/rgb24_prof.py 3 > /dev/null 2>&1; echo "k5u8f rc=$?"
timeout 300 python scripts/rgb24_micro.py > gpurun_out/${TAG}_rgb24_micro.log 2>&1
ls gpurun_out | grep "^${TAG}"
