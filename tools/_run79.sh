set -u
O=gpurun_out
T=r02zzb
timeout 1500 python -m pytest tests -m gpu -q > $O/${T}_gputests.log 2>&1; echo "pytest rc=$?"; tail -2 $O/${T}_gputests.log
timeout 900 python bench.py > $O/${T}_bench.json 2> $O/${T}_bench.err; echo "bench rc=$?"; tail -2 $O/${T}_bench.err
timeout 900 compute-sanitizer --tool memcheck --error-exitcode 9 python -m pytest tests/test_geometry_gpu.py tests/test_frame_gpu.py -x -q > $O/${T}_memcheck.log 2>&1; echo "memcheck rc=$?"; tail -3 $O/${T}_memcheck.log
timeout 900 compute-sanitizer --tool racecheck --error-exitcode 9 python -m pytest tests/test_frame_gpu.py -x -q -k "ragged or golden" > $O/${T}_racecheck.log 2>&1; echo "racecheck rc=$?"; tail -3 $O/${T}_racecheck.log
