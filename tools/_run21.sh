set -u
O=gpurun_out
TAG=r02y
for k in k_claim k_commit_bulk k_commit_sweep k_find; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$k -s 3 -c 1 \
    -o $O/prof_${k}_$TAG -f python bench.py --steps 1 --warmup 3 --profile > $O/prof_${k}_$TAG.stdout 2>&1; echo "$k rc=$?"
  bash tools/ncu_export.sh $O/prof_${k}_$TAG.ncu-rep
done
