set -u
O=gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > $O/r02e_gputests.log 2>&1; echo "pytest rc=$?"; tail -3 $O/r02e_gputests.log
timeout 300 python tools/exp_dedup.py all 6 > $O/r02e_dedup.txt 2>&1; cat $O/r02e_dedup.txt
for w in c3 c4 c4f; do
  timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/r02e_launch_$w.csv python tools/exp_dedup.py $w 3 > /dev/null 2>&1
  python tools/ncu_sum.py $O/r02e_launch_$w.csv | head -12
done
timeout 300 ncu --set full --clock-control none --import-source on -k regex:k_voxel_claim -s 2 -c 1 -o $O/r02e_vclaim_c3 -f python tools/exp_dedup.py c3 3 > /dev/null 2>&1; echo c3 rc=$?
timeout 300 ncu --set full --clock-control none --import-source on -k regex:k_voxel_select -s 2 -c 1 -o $O/r02e_vsel_c3 -f python tools/exp_dedup.py c3 3 > /dev/null 2>&1; echo c3s rc=$?
timeout 300 ncu --set full --clock-control none --import-source on -k regex:k_voxel_claim -s 12 -c 1 -o $O/r02e_vclaim_c4 -f python tools/exp_dedup.py c4 3 > /dev/null 2>&1; echo c4 rc=$?
timeout 300 ncu --set full --clock-control none --import-source on -k regex:k_voxel_claim -s 12 -c 1 -o $O/r02e_vclaim_c4f -f python tools/exp_dedup.py c4f 3 > /dev/null 2>&1; echo c4f rc=$?
ls -la $O
