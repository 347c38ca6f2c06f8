set -u
O=gpurun_out
timeout 300 python tools/exp_part_prof.py peer > $O/r02zs_part_peer.log 2>&1; echo rc=$?; tail -60 $O/r02zs_part_peer.log
