set -u
O=gpurun_out
timeout 600 python -m pytest tests/test_geometry_gpu.py -x -q > $O/r02zw_tests.log 2>&1; echo "tests rc=$?"; tail -3 $O/r02zw_tests.log
for G in 0 2 4 8 0 4; do echo "pipe=$G"; ASH_DD_PIPE=$G timeout 300 python tools/exp_dedup.py c3 10 2>&1 | grep "c3"; done
