set -u
O=gpurun_out
timeout 900 python -m pytest tests/test_geometry_gpu.py tests/test_device_len_gpu.py tests/test_frame_gpu.py tests/test_blocks_gpu.py -x -q > $O/r02zv_tests.log 2>&1; echo "tests rc=$?"; tail -3 $O/r02zv_tests.log
for L in 1 0 1 0; do echo "lookback=$L"; ASH_DD_LOOKBACK=$L timeout 300 python tools/exp_dedup.py all 8 2>&1 | grep -v "^\s*$" | tail -4; done
