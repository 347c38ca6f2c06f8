set -u
O=gpurun_out
T=r02zz8
timeout 1500 python -m pytest tests -m gpu -q > $O/${T}_gputests.log 2>&1; echo "pytest rc=$?"; tail -2 $O/${T}_gputests.log
timeout 900 python bench.py > $O/${T}_bench.json 2> $O/${T}_bench.err; echo "bench rc=$?"; tail -2 $O/${T}_bench.err
timeout 900 python bench.py --impl reference > $O/${T}_reference_arm.json 2> $O/${T}_reference_arm.err; echo "ref rc=$?"
timeout 600 python bench.py --partitioned > $O/${T}_partitioned_n1.json 2> $O/${T}_partitioned_n1.err; echo "part rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_${T}.csv python bench.py --steps 2 --warmup 3 --profile > /dev/null 2>&1; echo "launches rc=$?"
timeout 300 ncu --set full --clock-control none --import-source on -k regex:k_dd_claim_cloud -s 2 -c 1 -o $O/${T}_cloud_claim -f python tools/exp_dedup.py c3 3 > /dev/null 2>&1; echo "ncu cloud rc=$?"
