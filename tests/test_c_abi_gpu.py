"""The C ABI used from C alone (tests/c_abi/ash_c_client.c): cudaMalloc'd
buffers, ash_map_reset / ash_insert / activate / ash_erase / ash_find /
ash_active_indices, the generic-backend contract checked in the client."""
import subprocess

import pytest

from test_abi_cpu import build_c_client

pytestmark = pytest.mark.gpu


def test_plain_c_client_runs(cuda_ok, tmp_path):
    exe = build_c_client(tmp_path)
    r = subprocess.run([str(exe)], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stderr
    assert "ash_c_client OK" in r.stdout
