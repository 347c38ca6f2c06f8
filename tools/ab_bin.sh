#!/usr/bin/env bash
# A/B: slot-state commit by random stores vs table sweep (GPU box)
set -u
mkdir -p gpurun_out
timeout 600 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_ab.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_ab.log
for d in ${DIVS:-0 2}; do
  ASH_BIN_DIV=$d timeout 200 python bench.py --no-cpu-baseline > gpurun_out/ab_bin_$d.json 2> gpurun_out/ab_bin_$d.err
  python - "$d" <<'PY'
import json, sys
m = sys.argv[1]
try:
    d = json.loads(open(f"gpurun_out/ab_bin_{m}.json").read().strip().splitlines()[-1])
    print(f"div={m} value={d['value']} ms={d['ms_per_step']} kernels={d['roofline']['kernel_ms']} e2e={d['e2e']['value']}")
    print("  sweep", [(s['rho'], s['value'], s['insert_mops']) for s in d['sweep']])
except Exception as e:
    print(f"div={m} FAILED {e}"); print(open(f"gpurun_out/ab_bin_{m}.err").read()[-2000:])
PY
done
