set -u
O=gpurun_out
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/r02zc_launch_part.csv python bench.py --partitioned --steps 2 --warmup 3 --no-c5 > /dev/null 2>&1; echo rc=$?
python - <<PY
import csv
rows=list(csv.reader(open("$O/r02zc_launch_part.csv")))
h=next(i for i,r in enumerate(rows) if 'Kernel Name' in r)
H=rows[h]; ki=H.index('Kernel Name'); vi=H.index('Metric Value')
L=[(r[ki][:60], float(r[vi].replace(',',''))/1000) for r in rows[h+1:]]
# print the last ~45 launches (one step: insert + find)
for n,v in L[-60:]: print(f"{v:8.1f}  {n}")
PY
