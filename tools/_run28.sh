set -u
O=gpurun_out
timeout 300 python -m pytest tests/test_frame_gpu.py tests/test_device_len_gpu.py tests/test_parity_gpu.py -x -q > $O/r02zi_tests.log 2>&1; echo "tests rc=$?"; grep -E "passed|failed" $O/r02zi_tests.log | tail -2
timeout 300 python tools/exp_dedup.py all 8 2>&1 | tail -1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/r02zi_launch_c4.csv python tools/exp_dedup.py c4 3 > /dev/null 2>&1
python tools/ncu_sum.py $O/r02zi_launch_c4.csv 2>/dev/null | head -6
