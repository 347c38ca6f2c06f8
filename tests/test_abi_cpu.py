"""CPU-side checks of the C ABI library: it loads, exports every symbol the
header declares, and its struct layout matches the ctypes mirror.  No
compute calls (there is no GPU here)."""
import re
import subprocess
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
HEADER = ROOT / "include" / "ash.h"


def _declared():
    text = HEADER.read_text()
    return sorted(set(re.findall(r"^(?:int|int64_t|const char\*)\s+(ash_\w+)\(", text, re.M)))


def test_library_loads_and_exports_all_declared_symbols():
    from paper_2110_00511_b200 import _lib
    names = _declared()
    assert len(names) >= 15
    for n in names:
        assert hasattr(_lib.lib, n), f"libash.so does not export {n}"
    assert set(names) == set(_lib.EXPORTED), "ctypes signatures out of sync with ash.h"
    assert _lib.lib.ash_abi_version() == 7


def test_struct_layout_matches_header(tmp_path):
    from paper_2110_00511_b200 import _lib
    src = tmp_path / "sz.c"
    src.write_text(
        '#include <stdio.h>\n#include <stddef.h>\n#include "ash.h"\n'
        'int main(){printf("%zu %zu %zu %zu\\n", sizeof(ash_map_t), offsetof(ash_map_t, heap),'
        ' offsetof(ash_map_t, scan_status_len), offsetof(ash_map_t, epoch));return 0;}\n')
    exe = tmp_path / "sz"
    subprocess.run(["gcc", "-I", str(ROOT / "include"), str(src), "-o", str(exe)], check=True)
    got = list(map(int, subprocess.run([str(exe)], capture_output=True, text=True).stdout.split()))
    S = _lib.AshMap
    assert got == [_lib.ctypes.sizeof(S), S.heap.offset, S.scan_status_len.offset, S.epoch.offset]


def test_scan_tiles_and_error_plumbing():
    from paper_2110_00511_b200 import _lib
    assert _lib.scan_tiles(1) == 1
    assert _lib.scan_tiles(_lib.TILE) == 1
    assert _lib.scan_tiles(_lib.TILE + 1) == 2
    for n in (0, 1, 2047, 2048, 2049, 10_000_000, 2 ** 31):
        assert _lib.scan_tiles(n) == int(_lib.lib.ash_scan_tiles(n)), n
    # invalid arguments are rejected before any device work
    with pytest.raises(ValueError, match="null map"):
        _lib.call("ash_find", None, None, 0, None, None, None)
    with pytest.raises(ValueError, match="cell size"):
        _lib.call("ash_quantize", None, 1, 10, -1.0, None, None, None)


def test_no_oracle_import_in_product():
    pkg = ROOT / "paper_2110_00511_b200"
    for f in pkg.rglob("*.py"):
        assert "oracle" not in f.read_text().replace("oracle/", ""), f"{f} references the oracle"


def build_c_client(out_dir: Path) -> Path:
    """Compile tests/c_abi/ash_c_client.c (a plain C caller of ash.h) against
    libash.so and the CUDA runtime; warnings are errors."""
    cuda = Path("/usr/local/cuda")
    lib_dir = ROOT / "paper_2110_00511_b200" / "lib"
    exe = out_dir / "ash_c_client"
    subprocess.run(["gcc", "-std=c99", "-Wall", "-Wextra", "-Werror", "-I", str(ROOT / "include"),
                    "-I", str(cuda / "include"), str(ROOT / "tests" / "c_abi" / "ash_c_client.c"),
                    "-L", str(lib_dir), "-lash", "-L", str(cuda / "lib64"), "-lcudart",
                    f"-Wl,-rpath,{lib_dir}", "-o", str(exe)], check=True)
    return exe


def test_plain_c_client_compiles_and_links(tmp_path):
    """The header is plain C and a C caller links against the exports (the
    client itself runs in tests/test_c_abi_gpu.py)."""
    assert build_c_client(tmp_path).exists()
