set -u
O=gpurun_out
timeout 900 python -m pytest tests/test_peer_gpu.py tests/test_route_gpu.py -x -q 2>&1 | tail -3
timeout 300 python tools/exp_partition.py peer 2>&1 | grep -v Warn | tail -8
timeout 600 python bench.py --partitioned --steps 10 --warmup 3 2>&1 | tail -1
timeout 600 python bench.py --partitioned --transport nccl --steps 10 --warmup 3 2>&1 | tail -1
