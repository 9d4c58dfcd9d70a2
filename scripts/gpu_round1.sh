mkdir -p gpurun_out
set -x
nvidia-smi --query-gpu=name,memory.total,clocks.max.sm --format=csv
nproc; free -g
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"
tail -5 gpurun_out/smoke.log
timeout 600 python -m pytest tests/test_gpu_golden.py -x -q > gpurun_out/golden.log 2>&1; echo "golden rc=$?"
tail -30 gpurun_out/golden.log
timeout 300 python bench.py --steps 3 --warmup 2 --streams 16 --no-cpu-baseline --e2e-streams 4 > gpurun_out/bench1.log 2>&1; echo "bench rc=$?"
tail -5 gpurun_out/bench1.log
