set -u
O=gpurun_out
cap() {  # name regex skip script args...
  local name=$1 rx=$2 skip=$3; shift 3
  timeout 300 ncu --set full --clock-control none --import-source on -k regex:$rx -s $skip -c 1 -o $O/$name -f "$@" > /dev/null 2>&1
  echo "$name rc=$?"; bash tools/ncu_export.sh $O/$name.ncu-rep
}
timeout 600 python -m pytest tests/test_geometry_gpu.py tests/test_frame_gpu.py tests/test_device_len_gpu.py -x -q 2>&1 | tail -1
timeout 300 python tools/exp_dedup.py all 8 2>&1 | tail -3
cap r02q_emit_c3 k_dd_emit 2 python tools/exp_dedup.py c3 4
cap r02q_claim_c3 k_dd_claim 2 python tools/exp_dedup.py c3 4
