set -u
O=gpurun_out
timeout 600 python -m pytest tests/test_device_len_gpu.py -x -q 2>&1 | grep -E "passed|failed" | tail -1
timeout 900 compute-sanitizer --tool memcheck python -m pytest tests/test_device_len_gpu.py tests/test_route_gpu.py -x -q -k "not shared" > $O/san2.log 2>&1; echo "memcheck rc=$?"; grep -E "ERROR SUMMARY|passed|failed" $O/san2.log | tail -3
