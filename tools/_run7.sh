set -u
O=gpurun_out
timeout 300 python tools/exp_c4_host.py 2>&1 | tail -12
timeout 300 python tools/exp_dedup.py c4 6 2>&1 | tail -2
timeout 600 python -m pytest tests/test_device_len_gpu.py tests/test_frame_gpu.py tests/test_parity_gpu.py tests/test_fullsize_gpu.py -x -q 2>&1 | tail -2
