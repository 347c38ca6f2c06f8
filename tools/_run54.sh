set -u
O=gpurun_out
timeout 300 ncu --set full --clock-control none --import-source on -k regex:k_route_count -s 4 -c 1 -o $O/prof_k_route_count_r02zzc -f python tools/exp_count.py > /dev/null 2>&1; echo rc=$?
bash tools/ncu_export.sh $O/prof_k_route_count_r02zzc.ncu-rep
