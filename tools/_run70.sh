set -u
for D in 0 4 8 16; do echo "sparse_div=$D"; ASH_SPARSE_DIV=$D timeout 600 python tools/exp_spec.py 2>&1 | grep "spec=1" | awk 'NR%2==1'; done
