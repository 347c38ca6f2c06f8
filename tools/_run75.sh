set -u
# configs[2] cloud claim: L2 bulk prefetch distance sweep (ASH_CLOUD_PF, points ahead)
O=gpurun_out
for r in 1 2; do for pf in 0 75000 150000 300000 600000 1200000; do
  echo "pf=$pf $(ASH_CLOUD_PF=$pf timeout 300 python tools/exp_dedup.py c3 10 2>&1 | grep 'c3 voxelize' | sed 's/.*median/median/')"
done; done > $O/r02zz9_cloud_pf.txt 2>&1
cat $O/r02zz9_cloud_pf.txt
ASH_CLOUD_PF=300000 timeout 600 python -m pytest tests/test_geometry_gpu.py tests/test_fullsize_gpu.py -x -q 2>&1 | tail -2
