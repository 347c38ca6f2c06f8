"""Per-kernel totals of an ncu gpu__time_duration launch list (CSV):
    python tools/ncu_sum.py gpurun_out/launches.csv"""
import csv, sys
from collections import defaultdict
rows = list(csv.reader(open(sys.argv[1])))
h = next(i for i, r in enumerate(rows) if 'Kernel Name' in r)
H = rows[h]; ki = H.index('Kernel Name'); vi = H.index('Metric Value'); ii = H.index('ID')
agg = defaultdict(lambda: [0, 0.0])
for r in rows[h + 1:]:
    agg[r[ki][:60]][0] += 1
    agg[r[ki][:60]][1] += float(r[vi].replace(',', '')) / 1e3
tot = sum(v[1] for v in agg.values())
print(f"total {tot:.0f} us")
for k, v in sorted(agg.items(), key=lambda kv: -kv[1][1])[:14]:
    print(f"{v[1]:9.0f} us {v[0]:4d}x  {k}")
