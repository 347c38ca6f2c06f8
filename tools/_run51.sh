set -u
for D in 0 150000 300000 600000 1200000 0 300000; do
  ASH_PF_CLAIM=$D ASH_PF_FIND=$D timeout 300 python tools/exp_pf.py 2>&1 | tail -1
done
