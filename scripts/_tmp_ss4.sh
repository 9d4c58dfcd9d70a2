cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_pipeline.py tests/test_gpu_golden.py tests/test_gpu_api.py tests/test_gpu_residual.py -x -q -p no:cacheprovider 2>&1 | tail -3
timeout -s KILL 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
   --log-file gpurun_out/r02_ss3_launches.csv python scripts/single_stream_step.py 8 > /dev/null 2>&1
python scripts/launch_summary.py gpurun_out/r02_ss3_launches.csv 8 4
python - <<'PY'
import sys, json, types
sys.path.insert(0, ".")
import torch, bench
a = types.SimpleNamespace(height=1080, width=1920, drop=0.1)
print(json.dumps(bench.single_stream_latency(a, torch.device("cuda", 0))))
PY
