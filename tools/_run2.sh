set -u
O=gpurun_out
cap() {  # name regex skip script args...
  local name=$1 rx=$2 skip=$3; shift 3
  timeout 300 ncu --set full --clock-control none --import-source on -k regex:$rx -s $skip -c 1 -o $O/$name -f "$@" > /dev/null 2>&1
  echo "$name rc=$?"; bash tools/ncu_export.sh $O/$name.ncu-rep
}
cap r02f_vclaim_c3 k_voxel_claim 2 python tools/exp_dedup.py c3 3
cap r02f_vsel_c3 k_voxel_select 2 python tools/exp_dedup.py c3 3
cap r02f_vclaim_c4 k_voxel_claim 12 python tools/exp_dedup.py c4 3
cap r02f_vclaim_c4f k_voxel_claim 12 python tools/exp_dedup.py c4f 3
timeout 300 python tools/exp_partition.py peer > $O/r02f_partition_peer.txt 2>&1; cat $O/r02f_partition_peer.txt | tail -30
du -sh $O
