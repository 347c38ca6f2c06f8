set -u
O=gpurun_out
cap() {  # name regex skip script args...
  local name=$1 rx=$2 skip=$3; shift 3
  timeout 300 ncu --set full --clock-control none --import-source on -k regex:$rx -s $skip -c 1 -o $O/$name -f "$@" > /dev/null 2>&1
  echo "$name rc=$?"; bash tools/ncu_export.sh $O/$name.ncu-rep
}
cap r02h_harvest_c3 k_dd_harvest 1 python tools/exp_dedup.py c3 3
cap r02h_claim_c3 k_dd_claim 1 python tools/exp_dedup.py c3 3
cap r02h_select_c3 k_dd_select 1 python tools/exp_dedup.py c3 3
du -sh $O
