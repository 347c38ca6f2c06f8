set -u
O=gpurun_out

ASH_SHARED_GPU=1 timeout 600 python bench.py --gpus 2 --steps 3 --warmup 3 --no-c5 > $O/r02za_part2.json 2> $O/r02za_part2.err; echo "part2 rc=$?"; tail -c 1500 $O/r02za_part2.json

