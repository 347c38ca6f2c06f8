set -u
# A/B: two-group cp.async cloud claim (ASH_CLOUD_G2=1) vs the one-group claim
O=gpurun_out
for r in 1 2 3; do for g in 0 1; do
  echo "g2=$g $(ASH_CLOUD_G2=$g timeout 300 python tools/exp_dedup.py c3 12 2>&1 | grep 'c3 voxelize' | sed 's/.*median/median/')"
done; done > $O/r02zzc_cloud_g2.txt 2>&1
cat $O/r02zzc_cloud_g2.txt
ASH_CLOUD_G2=1 timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/r02zzc_g2_1.csv python tools/exp_dedup.py c3 4 > /dev/null 2>&1
ASH_CLOUD_G2=0 timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/r02zzc_g2_0.csv python tools/exp_dedup.py c3 4 > /dev/null 2>&1
for g in 0 1; do echo "ncu g2=$g"; python tools/ncu_sum.py $O/r02zzc_g2_$g.csv 2>/dev/null | head -3; done
ASH_CLOUD_G2=1 timeout 600 python -m pytest tests/test_geometry_gpu.py tests/test_fullsize_gpu.py -x -q 2>&1 | tail -2
ASH_CLOUD_G2=1 timeout 300 python tools/fuzz_quant.py 20000 20400 2>&1 | tail -1
