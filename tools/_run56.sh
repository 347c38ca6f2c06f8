set -u
O=gpurun_out
CS=/usr/local/cuda/bin/compute-sanitizer
timeout 1500 $CS --tool memcheck --print-limit 20 python -m pytest tests/test_spec_claim_gpu.py tests/test_lazy_commit_gpu.py -x -q > $O/r02zzs_memcheck_spec.log 2>&1; echo "memcheck spec rc=$?"; tail -4 $O/r02zzs_memcheck_spec.log
timeout 1500 $CS --tool memcheck --print-limit 20 python -m pytest tests/test_route_gpu.py -x -q -k "exchange or put or world1" > $O/r02zzs_memcheck_route.log 2>&1; echo "memcheck route rc=$?"; tail -4 $O/r02zzs_memcheck_route.log
timeout 1500 $CS --tool racecheck --print-limit 20 python -m pytest tests/test_route_gpu.py -x -q -k "device_count_matrix" > $O/r02zzs_racecheck_put.log 2>&1; echo "racecheck put rc=$?"; tail -4 $O/r02zzs_racecheck_put.log
