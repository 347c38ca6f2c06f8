set -u
O=gpurun_out
T=r02zzh
timeout 1500 python -m pytest tests -m gpu -q > $O/${T}_gputests.log 2>&1; echo "pytest rc=$?"; tail -2 $O/${T}_gputests.log
timeout 900 python bench.py > $O/${T}_bench.json 2> $O/${T}_bench.err; echo "bench rc=$?"; tail -2 $O/${T}_bench.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_${T}.csv python bench.py --steps 2 --warmup 3 --profile > /dev/null 2>&1; echo "launches rc=$?"
timeout 900 python tools/fuzz_ops.py 40000 40600 2>&1 | tail -1
