set -u
O=gpurun_out
timeout 900 python -m pytest tests/test_geometry_gpu.py tests/test_frame_gpu.py tests/test_device_len_gpu.py tests/test_parity_gpu.py -x -q > $O/r02ze_tests.log 2>&1; echo "tests rc=$?"; grep -E "passed|failed" $O/r02ze_tests.log | tail -2
timeout 300 python tools/exp_dedup.py all 8 2>&1 | tail -3
