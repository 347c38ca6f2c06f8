set -u
O=gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > $O/r02zzg_gputests.log 2>&1; echo "pytest rc=$?"; tail -2 $O/r02zzg_gputests.log
timeout 900 python bench.py --no-sweep > $O/r02zzg_bench.json 2> $O/r02zzg_bench.err; echo "bench rc=$?"
python - <<PY
import json
d=json.loads(open("$O/r02zzg_bench.json").read().strip().splitlines()[-1])
o=d['other_configs']
print(d['value'], d['step_time']['median_ms'], 'c1', o['c1']['median_ms'], 'c3', o['c3_voxelize']['ms'], 'c4', o['c4_allocate_blocks']['ms_per_frame'], o['c4_frame_fused']['ms_per_frame'], 'c5', o['c5_stream_1gpu']['ms_total'])
PY
ASH_SWEEP_TABLE_MIN=0 timeout 600 python tools/fuzz_ops.py 20000 20400 2>&1 | tail -1
timeout 600 python tools/fuzz_ops.py 30000 30400 2>&1 | tail -1
