#!/bin/bash
# Last evidence run of round 2: full GPU tests, smoke, the default bench,
# the int8 learned path's launch list and a --set full capture of K5-9.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
TAG=${1:-r02s5}
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/${TAG}_gputest.log 2>&1
echo "pytest rc=$?"; tail -2 gpurun_out/${TAG}_gputest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1; echo "smoke rc=$?"
timeout 1200 python bench.py > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err; echo "bench rc=$?"
timeout -s KILL 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:^k_ --csv \
   --log-file gpurun_out/${TAG}_learned_launches.csv python scripts/learned_step.py 32 2 i8 > /dev/null 2>&1
echo "learned launches rc=$?"
timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:k_upscale9f -s 1 -c 1 \
    -o gpurun_out/${TAG}_k_upscale9f python scripts/learned_step.py 32 2 i8 > /dev/null 2>&1; echo "k59 rc=$?"
ls gpurun_out | grep "^${TAG}"
