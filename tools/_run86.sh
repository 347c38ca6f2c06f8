set -u
O=gpurun_out
T=r02zzh
timeout 900 python bench.py --impl reference > $O/${T}_reference_arm.json 2> $O/${T}_reference_arm.err; echo "ref rc=$?"
timeout 600 python bench.py --partitioned > $O/${T}_partitioned_n1.json 2> $O/${T}_partitioned_n1.err; echo "part rc=$?"
