set -u
for S in 1 0; do echo "staged=$S"; ASH_PUT_STAGED=$S timeout 300 python tools/exp_put.py 2>&1 | tail -4; done
timeout 600 python -m pytest tests/test_route_gpu.py tests/test_peer_gpu.py -x -q 2>&1 | tail -3
ASH_PUT_STAGED=1 timeout 600 python bench.py --partitioned --no-c5 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('part', d['value'], d['step_time'])"
