set -u
O=gpurun_out
timeout 900 python -m pytest tests/test_geometry_gpu.py tests/test_parity_gpu.py tests/test_fullsize_gpu.py -x -q > $O/r02zd_tests.log 2>&1; echo "tests rc=$?"; grep -E "passed|failed" $O/r02zd_tests.log | tail -2
timeout 300 python tools/exp_dedup.py c3 10 2>&1 | tail -1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/r02zd_launch_c3.csv python tools/exp_dedup.py c3 4 > /dev/null 2>&1
python - <<PY
import csv
rows=list(csv.reader(open("$O/r02zd_launch_c3.csv")))
h=next(i for i,r in enumerate(rows) if 'Kernel Name' in r)
H=rows[h]; ki=H.index('Kernel Name'); vi=H.index('Metric Value')
print([ (r[ki][15:40], int(float(r[vi].replace(',',''))/1000)) for r in rows[h+1:]][-7:])
PY
