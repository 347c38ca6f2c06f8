set -u
for i in 1 2; do timeout 300 python tools/exp_dedup.py c4 10 2>&1 | grep "c4 allocate_blocks"; done
timeout 900 python -m pytest tests/test_geometry_gpu.py tests/test_device_len_gpu.py tests/test_frame_gpu.py tests/test_fullsize_gpu.py -x -q 2>&1 | tail -1
timeout 600 python tools/fuzz_dedup.py 3000 3100 2>&1 | tail -1
