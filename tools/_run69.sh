set -u
timeout 600 python tools/exp_spec.py 2>&1 | grep "spec=1"
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -1
timeout 600 python tools/fuzz_ops.py 80000 80400 2>&1 | tail -1
