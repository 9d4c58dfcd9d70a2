cd $GRAFT_REPO_ROOT
for k in k_packetize k_topk; do
timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:$k -s 4 -c 1 \
   -o gpurun_out/r02_ss_$k python scripts/single_stream_step.py 8 > /dev/null 2>&1
done
ls gpurun_out
