set -u
O=gpurun_out
T=r02zz2
timeout 900 python bench.py > $O/${T}_bench.json 2> $O/${T}_bench.err; echo "bench rc=$?"; tail -2 $O/${T}_bench.err
timeout 600 python bench.py --partitioned > $O/${T}_partitioned_n1.json 2> $O/${T}_partitioned_n1.err; echo "part rc=$?"
