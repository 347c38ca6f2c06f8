set -u
O=gpurun_out
timeout 600 python -m pytest tests/test_route_gpu.py tests/test_peer_gpu.py -x -q > $O/r02zz6_route_tests.log 2>&1; echo "route tests rc=$?"; tail -3 $O/r02zz6_route_tests.log
for S in 1 0; do echo "ASH_PULL_STAGED=$S"; ASH_PULL_STAGED=$S timeout 300 python tools/exp_put.py 2>&1 | grep -v "^$"; done > $O/r02zz6_pull_ab.txt; cat $O/r02zz6_pull_ab.txt
