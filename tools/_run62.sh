set -u
for i in 1 2; do timeout 300 python tools/exp_pf.py 2>&1 | tail -1; done
timeout 300 python tools/exp_step_prof.py 2>&1 | grep -v Warn | grep "tile_scan\|step after"
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -1
timeout 600 python tools/fuzz_ops.py 40000 40300 2>&1 | tail -1
