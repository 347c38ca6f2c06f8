"""The reference arm of bench.py runs on CPU only: its JSON line follows the
driver contract (impl, metric, value, cpu_baseline with cores, e2e)."""
import json
import os
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent


def test_reference_arm_json_contract():
    env = dict(os.environ, ASH_CPU_SAMPLE_KEYS="20000", CUDA_VISIBLE_DEVICES="")
    out = subprocess.run([sys.executable, "bench.py", "--impl", "reference", "--steps", "2", "--warmup", "3"],
                         cwd=ROOT, env=env, capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    d = json.loads(out.stdout.strip().splitlines()[-1])
    assert d["impl"] == "reference" and d["metric"] == "insert & find Mops/s (int3 keys)"
    assert d["unit"] == "Mops/s" and d["higher_is_better"] is True and d["value"] > 0
    assert d["cpu_baseline"]["cores"] == len(os.sched_getaffinity(0)) and d["cpu_baseline"]["kind"] == "port"
    assert d["e2e"]["value"] == d["value"] and d["e2e"]["h2d_bytes_per_step"] == 0
    assert d["steps"] == 2 and d["warmup"] == 3


def test_key_hash_shards_are_exact_maps():
    """Every copy of a key lands in one shard, in batch order: per-shard
    first occurrences are the global first occurrences."""
    sys.path.insert(0, str(ROOT))
    import numpy as np
    import bench
    from oracle.ash_oracle import OracleMap
    rng = np.random.default_rng(2)
    pool = rng.integers(-500, 500, size=(4000, 3)).astype(np.int32)
    keys = pool[rng.integers(0, len(pool), size=12000)]
    vals = rng.random((len(keys), 1), dtype=np.float32)
    whole = OracleMap(len(keys), 3, [np.float32]).insert(keys, vals).masks
    shards = bench._owner_shards(keys, vals, 5)
    assert sum(len(k) for k, _ in shards) == len(keys)
    assert sum(int(OracleMap(max(len(k), 1), 3, [np.float32]).insert(k, v).masks.sum()) for k, v in shards) == \
        int(whole.sum())
