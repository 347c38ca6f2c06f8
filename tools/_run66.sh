set -u
O=gpurun_out
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/r02zzh_launch_c4f.csv python tools/exp_dedup.py c4f 3 > /dev/null 2>&1; echo ncu rc=$?
python - <<'PY'
import csv, collections
rows=[r for r in csv.reader(open("gpurun_out/r02zzh_launch_c4f.csv")) if len(r)>10]
h=rows[0]; ki=h.index('Kernel Name'); vi=h.index('Metric Value')
agg=collections.defaultdict(list)
for r in rows[1:]:
    agg[r[ki][:60]].append(float(r[vi].replace(',',''))/1e3)
for k,v in sorted(agg.items(), key=lambda kv:-sum(kv[1])):
    print(f"{sum(v):8.1f} us {len(v):4d}x  med {sorted(v)[len(v)//2]:6.1f}  {k}")
PY
