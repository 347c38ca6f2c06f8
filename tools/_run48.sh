set -u
timeout 300 python tools/exp_dedup.py c4 8 2>&1 | grep c4
timeout 300 python tools/exp_host_cost.py 100000 2>&1 | head -1
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
