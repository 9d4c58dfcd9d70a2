cd $GRAFT_REPO_ROOT
timeout -s KILL 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
   --log-file gpurun_out/r02_ss_launches.csv python scripts/single_stream_step.py 8 > /dev/null 2>&1
python scripts/launch_summary.py gpurun_out/r02_ss_launches.csv 8 4
