set -u
O=gpurun_out
timeout 600 python -m pytest tests/test_peer_gpu.py tests/test_route_gpu.py -x -q > $O/r02zb_tests.log 2>&1; echo "tests rc=$?"; grep -E "passed|failed" $O/r02zb_tests.log | tail -2
timeout 600 python bench.py --partitioned --steps 10 --warmup 3 --no-c5 2>/dev/null | tail -1 | cut -c1-180
ASH_PEER_DN=0 timeout 600 python bench.py --partitioned --steps 10 --warmup 3 --no-c5 2>/dev/null | tail -1 | cut -c1-180
ASH_SHARED_GPU=1 timeout 600 python bench.py --gpus 2 --steps 3 --warmup 3 --no-c5 2>/dev/null | tail -1 | cut -c1-180
