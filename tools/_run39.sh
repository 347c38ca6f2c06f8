set -u
O=gpurun_out
timeout 300 python tools/exp_c4_host.py > $O/r02zu_c4host.log 2>&1; echo rc=$?; tail -12 $O/r02zu_c4host.log
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/r02zu_launch_c4.csv python tools/exp_dedup.py c4 3 > /dev/null 2>&1; echo ncu rc=$?
python - <<'PY'
import csv, collections
rows=[r for r in csv.reader(open("gpurun_out/r02zu_launch_c4.csv")) if len(r)>10]
h=rows[0]; ki=h.index('Kernel Name'); vi=h.index('Metric Value'); ii=h.index('ID')
agg=collections.defaultdict(list)
for r in rows[1:]:
    agg[r[ki][:60]].append(float(r[vi].replace(',',''))/1e3)
tot=sum(sum(v) for v in agg.values())
print("total us", round(tot,1))
for k,v in sorted(agg.items(), key=lambda kv:-sum(kv[1])):
    print(f"{sum(v):8.1f} us {len(v):4d}x  med {sorted(v)[len(v)//2]:6.1f}  {k}")
PY
