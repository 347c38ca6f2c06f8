set -u
O=gpurun_out
timeout 300 ncu --set full --clock-control none --import-source on -k regex:k_claim -s 3 -c 1 -o $O/prof_k_claim_c1_r02zzd -f python tools/exp_step_prof.py 100000 > /dev/null 2>&1; echo rc=$?
bash tools/ncu_export.sh $O/prof_k_claim_c1_r02zzd.ncu-rep
