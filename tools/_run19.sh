set -u
O=gpurun_out
timeout 600 compute-sanitizer --tool memcheck --show-backtrace device --print-limit 5 python -m pytest tests/test_route_gpu.py -x -q -k world1 > $O/r02w_san.log 2>&1; echo "rc=$?"
grep -v "^frame #" $O/r02w_san.log | grep -B2 -A12 "Invalid" | head -60
