set -u
timeout 300 python tools/exp_count.py 2>&1 | tail -5
timeout 900 python -m pytest tests/test_route_gpu.py tests/test_peer_gpu.py tests/test_bench_gpu.py -x -q 2>&1 | tail -1
timeout 600 python bench.py --partitioned --no-c5 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('part', d['value'], d['step_time'])"
