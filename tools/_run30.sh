set -u
O=gpurun_out
timeout 300 python tools/exp_dedup.py c4 8 2>&1 | tail -1
timeout 300 python tools/exp_dedup.py c4f 8 2>&1 | tail -1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/r02zk_launch_c4f.csv python tools/exp_dedup.py c4f 3 > /dev/null 2>&1
python tools/ncu_sum.py $O/r02zk_launch_c4f.csv 2>/dev/null | head -4
