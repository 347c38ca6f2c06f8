set -u
O=gpurun_out
T=r02zz
for K in claim commit_bulk commit_sweep find; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_${K} -s 3 -c 1 -o $O/prof_k_${K}_${T} -f python bench.py --steps 2 --warmup 3 --profile > /dev/null 2>&1; echo "$K rc=$?"
  bash tools/ncu_export.sh $O/prof_k_${K}_${T}.ncu-rep
done
ls -la $O | grep prof_k | grep $T
