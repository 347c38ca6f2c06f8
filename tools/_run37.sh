set -u
O=gpurun_out
timeout 600 python -m pytest tests/test_route_gpu.py tests/test_peer_gpu.py -x -q > $O/r02zt_route.log 2>&1; echo "route rc=$?"; tail -15 $O/r02zt_route.log
timeout 300 python tools/exp_part_prof.py peer > $O/r02zt_part_peer.log 2>&1; echo rc=$?; grep -v "^frame\|^\[rank\|CUDA driver\|Exception raised\|^$" $O/r02zt_part_peer.log | tail -34
