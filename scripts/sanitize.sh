# compute-sanitizer memcheck / racecheck over small GPU tests
mkdir -p gpurun_out
CS=/usr/local/cuda/bin/compute-sanitizer
timeout -s KILL 900 $CS --tool memcheck --error-exitcode 9 --print-limit 20 python -m pytest tests/test_gpu_api.py -q -x -k "not 1080" > gpurun_out/san_api.log 2>&1; echo "memcheck api rc=$?"; tail -4 gpurun_out/san_api.log
timeout -s KILL 900 $CS --tool memcheck --error-exitcode 9 --print-limit 20 python -m pytest tests/test_gpu_pipeline.py -q -x -k "sweep or loss or corrupt" > gpurun_out/san_pipe.log 2>&1; echo "memcheck pipeline rc=$?"; tail -4 gpurun_out/san_pipe.log
timeout -s KILL 900 $CS --tool memcheck --error-exitcode 9 --print-limit 20 python -m pytest tests/test_gpu_learned.py -q -x -k "conv233 or attention or patchify or dec_in or fsq or pixels" > gpurun_out/san_learned.log 2>&1; echo "memcheck learned rc=$?"; tail -4 gpurun_out/san_learned.log
timeout -s KILL 900 $CS --tool racecheck --error-exitcode 9 --print-limit 20 python -m pytest tests/test_gpu_pipeline.py -q -x -k "sweep and 0" > gpurun_out/san_race.log 2>&1; echo "racecheck rc=$?"; tail -4 gpurun_out/san_race.log
timeout -s KILL 900 $CS --tool memcheck --error-exitcode 9 --print-limit 20 python -m pytest tests/test_gpu_upscale9.py -q -x -k "not 1080p" > gpurun_out/san_up9.log 2>&1; echo "memcheck upscale9 rc=$?"; tail -4 gpurun_out/san_up9.log
timeout -s KILL 900 $CS --tool racecheck --error-exitcode 9 --print-limit 20 python -m pytest tests/test_gpu_upscale9.py -q -x -k "blend and 50" > gpurun_out/san_race9.log 2>&1; echo "racecheck upscale9 rc=$?"; tail -4 gpurun_out/san_race9.log
timeout -s KILL 900 $CS --tool racecheck --error-exitcode 9 --print-limit 20 python -m pytest tests/test_gpu_learned.py -q -x -k "persistent_attention and 13" > gpurun_out/san_race_attn.log 2>&1; echo "racecheck attention rc=$?"; tail -4 gpurun_out/san_race_attn.log
