set -u
O=gpurun_out
timeout 300 python -m pytest tests/test_spec_claim_gpu.py -x -q > $O/r02zr_spec_tests.log 2>&1; echo "spec rc=$?"; tail -25 $O/r02zr_spec_tests.log
timeout 1200 python -m pytest tests -m gpu -x -q > $O/r02zr_gputests.log 2>&1; echo "pytest rc=$?"; tail -3 $O/r02zr_gputests.log
timeout 900 python bench.py > $O/r02zr_bench.json 2> $O/r02zr_bench.err; echo "bench rc=$?"; tail -3 $O/r02zr_bench.err
