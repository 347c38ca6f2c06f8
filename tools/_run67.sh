set -u
for i in 1 2; do timeout 300 python tools/exp_dedup.py c4 10 2>&1 | grep "c4 allocate_blocks" | sed 's/.*median/median/'; done
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_activate_small --csv --log-file gpurun_out/r02zzi_act.csv python tools/exp_dedup.py c4 2 > /dev/null 2>&1
python -c "
import csv
rows=[r for r in csv.reader(open('gpurun_out/r02zzi_act.csv')) if len(r)>10]
h=rows[0]; vi=h.index('Metric Value'); v=sorted(float(r[vi].replace(',',''))/1e3 for r in rows[1:]); print('activate_small median us', v[len(v)//2], len(v))"
timeout 900 python -m pytest tests/test_device_len_gpu.py tests/test_frame_gpu.py tests/test_geometry_gpu.py -x -q 2>&1 | tail -1
timeout 600 python tools/fuzz_dedup.py 7000 7100 2>&1 | tail -1
