set -u
for i in 1 2; do timeout 300 python tools/exp_pf.py 2>&1 | tail -1; done
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
