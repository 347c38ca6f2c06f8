#!/usr/bin/env bash
# A/B matrix over table load factor and L2 stream hints (GPU box).
mkdir -p gpurun_out
for f in ${FACTORS:-2.0 1.5 1.25}; do
  for h in ${HINTS:-1 0}; do
    ASH_TABLE_FACTOR=$f ASH_STREAM_HINTS=$h timeout 300 python bench.py --no-cpu-baseline > gpurun_out/exp_f${f}_h${h}.json 2>&1
    python - "$f" "$h" <<'EOF'
import json, sys
f, h = sys.argv[1:3]
try:
    d = json.loads(open(f"gpurun_out/exp_f{f}_h{h}.json").read().strip().splitlines()[-1])
    sw = {(s["rho"], s["value"]): (s["insert_mops"], s["find_mops"]) for s in d["sweep"]}
    print(f"factor={f} hints={h} value={d['value']} kernels={d['roofline']['kernel_ms']} "
          f"rho0.1={sw[(0.1,'f32[1]')]} rho1.0={sw[(1.0,'f32[1]')]} rho1.0x8={sw[(1.0,'f32[8]')]}")
except Exception as e:
    print(f"factor={f} hints={h} FAILED {e}")
    print(open(f"gpurun_out/exp_f{f}_h{h}.json").read()[-2000:])
EOF
  done
done
