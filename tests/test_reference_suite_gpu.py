"""The reference's OWN test files, run unmodified against the drop-in.

tests/reference_suite/spatialhash/ binds the name ``spatialhash`` to the
numpy-facing drop-in (``paper_2110_00511_b200.numpy_api``); the reference's
TSDF / bench / io / cli code and its ``spatialhash_arrays`` wrapper run from
the reference's own sources on top of the device map.  The reference files
are read from /root/reference (build container) or from the staged copy
baseline/_ref_suite (tools/stage_reference_suite.sh; the GPU box has no
/root/reference).  Skipped when neither exists.

Every collected reference test must pass except the ones listed in
DEVIATIONS, each with the documented reason."""
import json
import os
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu

ROOT = Path(__file__).resolve().parent.parent
STAGED = ROOT / "baseline" / "_ref_suite"

# reference test id -> why it cannot pass here (not a drop-in difference)
DEVIATIONS: dict = {
    "test_report_renders_figures": "needs matplotlib, which this image does not have (report "
                                   "plotting is out of scope, SURVEY §2)",
}


def _layout():
    if (STAGED / "tests").exists():
        return STAGED / "tests", STAGED / "pkg", STAGED / "bindings_tests", STAGED / "bindings"
    ref = Path("/root/reference/pkg")
    if ref.exists():
        return ref / "tests", ref / "src", ref / "bindings" / "tests", ref / "bindings" / "src"
    return None


def test_reference_suite_on_the_drop_in(cuda_ok, tmp_path):
    lay = _layout()
    if lay is None:
        pytest.skip("reference test files not available (run tools/stage_reference_suite.sh)")
    tests, pkg, btests, bsrc = lay
    report = tmp_path / "report.json"
    env = dict(os.environ, ASH_REF_PKG=str(pkg),
               PYTHONPATH=os.pathsep.join([str(ROOT / "tests" / "reference_suite"), str(bsrc), str(tests)]))
    code = (
        "import json, sys, pytest\n"
        "class R:\n"
        "    def __init__(self): self.out = {}\n"
        "    def pytest_runtest_logreport(self, report):\n"
        "        if report.when == 'call' or report.outcome != 'passed':\n"
        "            self.out.setdefault(report.nodeid, report.outcome)\n"
        "            if report.outcome == 'failed': self.out[report.nodeid] = 'failed'\n"
        "r = R()\n"
        f"rc = pytest.main(['-q', '-p', 'no:cacheprovider', '--rootdir', {str(tests.parent)!r}, "
        f"{str(tests)!r}, {str(btests)!r}], plugins=[r])\n"
        f"open({str(report)!r}, 'w').write(json.dumps(r.out))\n")
    proc = subprocess.run([sys.executable, "-c", code], env=env, cwd=str(tmp_path),
                          capture_output=True, text=True, timeout=1500)
    assert report.exists(), proc.stdout[-3000:] + proc.stderr[-3000:]
    out = json.loads(report.read_text())
    summary_dir = ROOT / "gpurun_out"
    if summary_dir.exists():
        (summary_dir / "reference_suite.json").write_text(json.dumps(out, indent=1))
        (summary_dir / "reference_suite.log").write_text(proc.stdout[-200000:])
    failed = sorted(k for k, v in out.items() if v == "failed" and not any(d in k for d in DEVIATIONS))
    passed = sum(1 for v in out.values() if v == "passed")
    assert not failed, f"{len(failed)} reference tests failed ({passed} passed): {failed[:40]}\n" + \
        proc.stdout[-5000:]
    assert passed > 200
