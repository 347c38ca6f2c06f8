set -u
O=gpurun_out
timeout 900 python -m pytest tests/test_peer_gpu.py tests/test_route_gpu.py tests/test_device_len_gpu.py tests/test_frame_gpu.py tests/test_parity_gpu.py -x -q > $O/r02u_tests.log 2>&1; echo "rc=$?"
grep -E "passed|failed|Error|error" $O/r02u_tests.log | tail -5
