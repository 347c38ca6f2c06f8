set -u
timeout 300 python tools/exp_dedup.py c3 10 2>&1 | grep c3
timeout 600 python -m pytest tests/test_geometry_gpu.py tests/test_fullsize_gpu.py -x -q 2>&1 | tail -2
