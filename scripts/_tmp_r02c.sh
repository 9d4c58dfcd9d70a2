cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_gpu_learned_i8.py tests/test_gpu_upscale9.py -x -q -p no:cacheprovider 2>&1 | tail -3
timeout -s KILL 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:^k_ --csv \
   --log-file gpurun_out/r02c_i8_launches.csv python scripts/learned_step.py 32 2 i8 > /dev/null 2>&1
python scripts/launch_summary.py gpurun_out/r02c_i8_launches.csv
