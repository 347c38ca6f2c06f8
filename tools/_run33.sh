set -u
O=gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > $O/r02zp_gputests.log 2>&1; echo "pytest rc=$?"; tail -3 $O/r02zp_gputests.log
timeout 900 python bench.py > $O/r02zp_bench.json 2> $O/r02zp_bench.err; echo "bench rc=$?"; tail -3 $O/r02zp_bench.err
