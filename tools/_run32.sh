set -u
O=gpurun_out
timeout 300 ncu --set full --clock-control none --import-source on -k regex:k_dd_claim_cloud -s 2 -c 1 -o $O/r02zn_claimc -f python tools/exp_dedup.py c3 4 > /dev/null 2>&1; echo rc=$?
bash tools/ncu_export.sh $O/r02zn_claimc.ncu-rep
