#!/usr/bin/env bash
# A/B: device insert chunk size (GPU box)
for c in ${CHUNKS:-0 4194304 2097152 1048576 524288 262144}; do
  ASH_INSERT_CHUNK=$c timeout 300 python bench.py --no-cpu-baseline > gpurun_out/chunk_$c.json 2>&1
  python - "$c" <<'PY'
import json, sys
c = sys.argv[1]
try:
    d = json.loads(open(f"gpurun_out/chunk_{c}.json").read().strip().splitlines()[-1])
    sw = {(s["rho"], s["value"]): s["insert_mops"] for s in d["sweep"]}
    print(f"chunk={c} value={d['value']} e2e={d['e2e']['value']} ins(0.1,0.5,1.0 f32[1])="
          f"{sw[(0.1,'f32[1]')]},{sw[(0.5,'f32[1]')]},{sw[(1.0,'f32[1]')]} f32[8]@1.0={sw[(1.0,'f32[8]')]} "
          f"c5={d['other_configs']['c5_stream_1gpu']['mops']} c5_ins_ms={d['other_configs']['c5_stream_1gpu']['insert_ms_first_last']}")
except Exception as e:
    print(f"chunk={c} FAILED {e}"); print(open(f"gpurun_out/chunk_{c}.json").read()[-1500:])
PY
done
