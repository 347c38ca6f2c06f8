#!/usr/bin/env bash
# binned-claim iteration: parity tests (forced on), A/B bench, per-kernel launch list
set -u
mkdir -p gpurun_out
timeout 300 python -m pytest -x -q tests/test_parity_gpu.py tests/test_fullsize_gpu.py > gpurun_out/pytest_bin.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_bin.log
for d in ${DIVS:-0 2}; do
  ASH_BIN_DIV=$d timeout 200 python bench.py --no-cpu-baseline > gpurun_out/ab_bin_$d.json 2> gpurun_out/ab_bin_$d.err
  python - "$d" <<'PY'
import json, sys
m = sys.argv[1]
try:
    d = json.loads(open(f"gpurun_out/ab_bin_{m}.json").read().strip().splitlines()[-1])
    print(f"div={m} value={d['value']} ms={d['ms_per_step']} kernels={d['roofline']['kernel_ms']}")
    print("  sweep", [(s['rho'], s['value'], s['insert_mops']) for s in d['sweep']])
except Exception as e:
    print(f"div={m} FAILED {e}"); print(open(f"gpurun_out/ab_bin_{m}.err").read()[-2000:])
PY
done
ASH_BIN_DIV=2 timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"k_bin|k_excl|k_region|k_claim_spill|k_tile_count" -c 6 --csv --log-file gpurun_out/bin_ncu.csv python bench.py --steps 1 --warmup 1 --profile > /dev/null 2>&1
python - <<'PY'
import csv
rows=[r for r in csv.reader(open('gpurun_out/bin_ncu.csv')) if r]
h=next(i for i,r in enumerate(rows) if 'Kernel Name' in r); H=rows[h]
ki,mi,vi=H.index('Kernel Name'),H.index('Metric Name'),H.index('Metric Value')
d={}
for r in rows[h+1:]:
    d.setdefault((int(r[0]), r[ki].split('(')[0][:40]),{})[r[mi]]=r[vi]
for (i,k),m in sorted(d.items()):
    print(i,k, m.get('gpu__time_duration.sum'), 'rd',m.get('dram__bytes_read.sum'),'wr',m.get('dram__bytes_write.sum'))
PY
