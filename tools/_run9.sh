set -u
O=gpurun_out
timeout 900 python -m pytest tests/test_geometry_gpu.py tests/test_parity_gpu.py tests/test_fullsize_gpu.py -x -q > $O/r02o_tests.log 2>&1; echo "pytest rc=$?"; tail -3 $O/r02o_tests.log
timeout 300 python tools/exp_dedup.py c3 8 2>&1 | tail -2
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/r02o_launch_c3.csv python tools/exp_dedup.py c3 3 > /dev/null 2>&1
python tools/ncu_sum.py $O/r02o_launch_c3.csv 2>/dev/null | head -12
