set -u
O=gpurun_out
for X in 1 0; do
ASH_PEER_XCHG=$X timeout 600 python bench.py --partitioned > $O/r02zt_part_x$X.json 2> $O/r02zt_part_x$X.err; echo "x$X rc=$?"
python - <<PY
import json
d=json.loads(open("$O/r02zt_part_x$X.json").read().strip().splitlines()[-1])
print("x$X", d["value"], d["step_time"], {k: (v.get("mops"), v.get("ms_total")) for k, v in d["other_configs"].items()})
PY
done
