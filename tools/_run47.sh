set -u
timeout 300 python tools/exp_dedup.py c4 8 2>&1 | grep c4
timeout 300 python tools/exp_c4_host.py 2>&1 | tail -8
timeout 900 python -m pytest tests/test_device_len_gpu.py tests/test_frame_gpu.py tests/test_geometry_gpu.py tests/test_tsdf_gpu.py -x -q 2>&1 | tail -2
