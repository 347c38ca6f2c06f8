set -u
O=gpurun_out
timeout 900 python -m pytest tests/test_peer_gpu.py tests/test_route_gpu.py tests/test_device_len_gpu.py tests/test_frame_gpu.py tests/test_parity_gpu.py -x -q 2>&1 | tail -3
timeout 300 python tools/exp_dedup.py c4 6 2>&1 | tail -2
timeout 600 python bench.py --partitioned --steps 10 --warmup 3 2>&1 | tail -1
