set -u
O=gpurun_out
for dn in 1; do
ASH_PEER_DN=$dn timeout 300 python -m pytest tests/test_route_gpu.py -x -q -k world1 > $O/r02v_$dn.log 2>&1; echo "dn=$dn rc=$?"
grep -v "^frame #" $O/r02v_$dn.log | grep -iE "passed|failed|error|abort|what\(\)|terminate" | head -8
done
timeout 900 python -m pytest tests/test_peer_gpu.py tests/test_route_gpu.py tests/test_device_len_gpu.py tests/test_frame_gpu.py tests/test_parity_gpu.py -x -q > $O/r02x_tests.log 2>&1; echo "rc=$?"
grep -v "^frame #" $O/r02x_tests.log | grep -E "passed|failed" | tail -3
timeout 600 python bench.py --partitioned --steps 10 --warmup 3 2>&1 | tail -1 | cut -c1-200
ASH_PEER_DN=0 timeout 600 python bench.py --partitioned --steps 10 --warmup 3 2>&1 | tail -1 | cut -c1-200
