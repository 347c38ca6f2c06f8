set -u
O=gpurun_out
timeout 900 python -m pytest tests/test_geometry_gpu.py tests/test_frame_gpu.py tests/test_device_len_gpu.py tests/test_parity_gpu.py -x -q 2>&1 | tail -2
for v in 0 12 16; do
  echo "variant $v"
  ASH_CLOUD_CLAIM=$v timeout 300 python tools/exp_dedup.py c3 10 2>&1 | tail -1
  ASH_CLOUD_CLAIM=$v timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/r02p_launch_c3_$v.csv python tools/exp_dedup.py c3 4 > /dev/null 2>&1
  python - <<PY
import csv
rows=list(csv.reader(open("$O/r02p_launch_c3_$v.csv")))
h=next(i for i,r in enumerate(rows) if 'Kernel Name' in r)
H=rows[h]; ki=H.index('Kernel Name'); vi=H.index('Metric Value')
print([ (r[ki][15:40], int(float(r[vi].replace(',',''))/1000)) for r in rows[h+1:] if 'dd_' in r[ki]][-4:])
PY
done
timeout 300 python tools/exp_dedup.py c4 6 2>&1 | tail -2
