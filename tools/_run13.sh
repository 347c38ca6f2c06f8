set -u
O=gpurun_out
for f in 4 3 2 1.5; do
  echo "factor $f"
  ASH_WS_FACTOR=$f timeout 300 python tools/exp_dedup.py c3 10 2>&1 | tail -1
done
ASH_WS_FACTOR=2 timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/r02s_launch_c3.csv python tools/exp_dedup.py c3 4 > /dev/null 2>&1
python tools/ncu_sum.py $O/r02s_launch_c3.csv 2>/dev/null | head -8
