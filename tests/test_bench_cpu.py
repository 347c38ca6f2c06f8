"""The reference arm of bench.py runs on CPU only: its JSON line follows the
driver contract (impl, metric, value, cpu_baseline with cores, e2e), uses
the GPU arm's config dict, and never maps libash.so."""
import json
import os
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent


def test_reference_arm_json_contract():
    env = dict(os.environ, ASH_BENCH_KEYS="20000", CUDA_VISIBLE_DEVICES="")
    out = subprocess.run([sys.executable, "bench.py", "--impl", "reference", "--steps", "2", "--warmup", "3"],
                         cwd=ROOT, env=env, capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    d = json.loads(out.stdout.strip().splitlines()[-1])
    assert d["impl"] == "reference" and d["metric"] == "insert & find Mops/s (int3 keys)"
    assert d["unit"] == "Mops/s" and d["higher_is_better"] is True and d["value"] > 0
    assert d["cpu_baseline"]["kind"] in ("reference", "port") and d["cpu_baseline"]["cores"] >= 1
    if (ROOT / "baseline" / "_ref" / "spatialhash").exists():
        assert d["cpu_baseline"]["kind"] == "reference"
    assert d["e2e"]["value"] == d["value"] and d["e2e"]["h2d_bytes_per_step"] == 0
    assert d["steps"] == 2 and d["warmup"] == 3 and d["step_time"]["trials"] == 2
    assert d["libash_mapped"] is False
    assert d["config"]["keys"] == 20000 and "gen_keys(20_000" in d["config"]["workload"]
    assert len(d["other_configs"]["sweep"]) == 6 and "threads=1" in d["other_configs"]["c1"]


def test_both_arms_share_the_config_dict():
    env = dict(os.environ, CUDA_VISIBLE_DEVICES="")
    code = ("import bench, json; print(json.dumps(bench.CONFIG))")
    out = subprocess.run([sys.executable, "-c", code], cwd=ROOT, env=env, capture_output=True, text=True)
    cfg = json.loads(out.stdout)
    assert cfg["keys"] == 10_000_000 and cfg["capacity"] == 10_000_000 and cfg["uniqueness"] == 0.5
    src = (ROOT / "bench.py").read_text()
    assert src.count('"config": CONFIG') == 2  # the GPU line and the reference line


def test_gen_keys_matches_reference_digests():
    """workloads.gen_keys is the reference generator output for output: the
    SHA-256 of its C1 and C2 batches equals the digests the reference wrote."""
    import hashlib
    import importlib.util
    spec = importlib.util.spec_from_file_location("wl", ROOT / "paper_2110_00511_b200" / "workloads.py")
    wl = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(wl)
    g = json.loads((ROOT / "tests" / "golden" / "fullsize_sha.json").read_text())
    for name, v in g["gen_keys"].items():
        a = wl.gen_keys(v["n"], v["rho"], "int3", v["seed"])
        assert hashlib.sha256(a.tobytes()).hexdigest() == v["sha"], name


def test_gen_keys_small_cases_match_reference():
    ref = Path("/root/reference/pkg/src")
    if not ref.exists():
        pytest.skip("reference not present (GPU box)")
    sys.path.insert(0, str(ref))
    import numpy as np
    from spatialhash.bench import gen_keys as ref_gen
    sys.path.insert(0, str(ROOT))
    from paper_2110_00511_b200.workloads import gen_keys
    for n, rho, kind, seed in [(1, 1.0, "int3", 0), (64, 0.5, "int3", 1), (1000, 0.37, "int3", 9),
                               (5000, 0.2, "int1", 4), (20000, 1.0, "int1", 5)]:
        assert np.array_equal(ref_gen(n, rho, kind, seed), gen_keys(n, rho, kind, seed)), (n, rho, kind)


def test_package_import_does_not_load_libash():
    code = ("import paper_2110_00511_b200 as p, paper_2110_00511_b200.workloads as w; "
            "from pathlib import Path; print('libash.so' in Path('/proc/self/maps').read_text())")
    out = subprocess.run([sys.executable, "-c", code], cwd=ROOT, capture_output=True, text=True)
    assert out.stdout.strip() == "False", out.stderr


def test_self_launch_runs_torchrun_on_localhost(monkeypatch):
    """`python bench.py --gpus N` without torchrun launches its own N ranks
    the way the driver does (torch.distributed.run, 127.0.0.1)."""
    import subprocess
    import sys
    import bench
    seen = {}
    monkeypatch.setattr(subprocess, "call", lambda cmd: seen.setdefault("cmd", cmd) and 0)
    monkeypatch.setattr(sys, "argv", ["bench.py", "--gpus", "4", "--steps", "3"])
    assert bench.self_launch(4) == 0
    cmd = seen["cmd"]
    assert cmd[1:3] == ["-m", "torch.distributed.run"]
    assert "--nproc-per-node=4" in cmd and "--master-addr=127.0.0.1" in cmd
    assert cmd[-3:] == ["--gpus", "4", "--steps", "3"][-3:] and cmd[-5].endswith("bench.py")
