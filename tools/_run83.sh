set -u
# A/B: table sweep writing whole 32-byte buckets (ASH_SWEEP_FULL=1) vs 4-byte state stores
O=gpurun_out
for r in 1 2; do for f in 0 1; do
  ASH_SWEEP_FULL=$f timeout 600 python bench.py --no-cpu-baseline > $O/r02zzg_sweep_$f$r.json 2> $O/r02zzg_sweep_$f$r.err
  python - "$f$r" <<'PY'
import json, sys
t = sys.argv[1]
d = json.loads(open(f"gpurun_out/r02zzg_sweep_{t}.json").read().strip().splitlines()[-1])
print(f"full={t[0]} run={t[1]} value={d['value']} ms={d['ms_per_step']} kernels={d['roofline']['kernel_ms']}")
print("  sweep", [(s['rho'], s.get('value_shape', s.get('shape')), s['insert_mops']) for s in d['sweep']][:6])
PY
done; done > $O/r02zzg_sweep_ab.txt 2>&1
cat $O/r02zzg_sweep_ab.txt
ASH_SWEEP_FULL=1 timeout 900 python -m pytest tests/test_parity_gpu.py tests/test_fullsize_gpu.py tests/test_lazy_commit_gpu.py tests/test_spec_claim_gpu.py tests/test_hashmap_gpu.py -x -q 2>&1 | tail -2
