set -u
for S in 1 0 1 0; do ASH_SWEEP_TMA=$S timeout 300 python tools/exp_pf.py 2>&1 | tail -1 | sed "s/^/tma=$S /"; done
timeout 900 python -m pytest tests/test_spec_claim_gpu.py tests/test_lazy_commit_gpu.py tests/test_parity_gpu.py tests/test_fullsize_gpu.py tests/test_hashmap_gpu.py -x -q 2>&1 | tail -1
