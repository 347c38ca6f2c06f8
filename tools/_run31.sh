set -u
O=gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > $O/r02zl_tests.log 2>&1; echo "tests rc=$?"; grep -E "passed|failed" $O/r02zl_tests.log | tail -2
timeout 600 python bench.py --no-sweep --no-cpu-baseline --steps 10 --warmup 3 > $O/r02zl_bench.json 2>/dev/null; python - <<PY
import json
d=json.loads(open("$O/r02zl_bench.json").read().strip().splitlines()[-1])
print(d["value"], d["ms_per_step"], {k:(v.get("median_ms") or v.get("ms") or v.get("ms_per_frame") or v.get("mops")) for k,v in d["other_configs"].items()})
PY
