"""bench.py's N-rank path end to end on one GPU: `ASH_SHARED_GPU=1 python
bench.py --gpus 2` launches two ranks itself (torch.distributed.run), both on
cuda:0 with a gloo control plane and CUDA-IPC peer mappings, and rank 0
prints one line for N = 2 with the configs[4] strong-scaling entry (shrunk
by ASH_C5_TOTAL to keep the test short).  A functional check of the
multi-rank bench, not a scaling number."""
import json
import os
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu

ROOT = Path(__file__).resolve().parent.parent


def test_bench_two_ranks_self_launched(cuda_ok):
    env = dict(os.environ, ASH_SHARED_GPU="1", ASH_C5_TOTAL="4000000")
    out = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--gpus", "2", "--steps", "2", "--warmup", "3"],
                         cwd=ROOT, env=env, capture_output=True, text=True, timeout=900)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert lines, out.stdout[-2000:]
    d = json.loads(lines[-1])
    assert d["n_gpus"] == 2 and d["scaling"] == "weak" and d["value"] > 0
    assert d["step_time"]["trials"] == 2 and d["e2e"]["value"] > 0 and d["clocks"]
    c5 = d["other_configs"]["c5_partitioned_peer"]
    assert c5["keys"] == 4_000_000 and c5["mops"] > 0 and c5["scaling"] == "strong"
