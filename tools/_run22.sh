set -u
O=gpurun_out
timeout 900 python bench.py --partitioned --steps 5 --warmup 3 > $O/r02z_part1.json 2> $O/r02z_part1.err; echo "part1 rc=$?"; tail -c 2500 $O/r02z_part1.json; grep -v "^frame\|Warn\|warn" $O/r02z_part1.err | tail -5
ASH_SHARED_GPU=1 timeout 1200 python bench.py --gpus 2 --steps 3 --warmup 3 > $O/r02z_part2.json 2> $O/r02z_part2.err; echo "part2 rc=$?"; tail -c 2500 $O/r02z_part2.json; grep -v "^frame\|Warn\|warn" $O/r02z_part2.err | tail -5
