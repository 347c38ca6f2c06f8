set -u
O=gpurun_out
timeout 900 python -m pytest tests/test_device_len_gpu.py tests/test_geometry_gpu.py tests/test_frame_gpu.py tests/test_parity_gpu.py tests/test_fullsize_gpu.py -x -q > $O/r02n_tests.log 2>&1; echo "pytest rc=$?"; tail -3 $O/r02n_tests.log
timeout 300 python tools/exp_c4_host.py 2>&1 | tail -9
timeout 300 python tools/exp_dedup.py all 6 2>&1 | tail -4
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/r02n_launch_c4.csv python tools/exp_dedup.py c4 3 > /dev/null 2>&1
python tools/ncu_sum.py $O/r02n_launch_c4.csv 2>/dev/null | head -14
