"""pytest plugin: run the REFERENCE's own test files against the drop-in.

Loaded with ``-p reference_alias`` before the reference's conftest.  It
registers ``spatialhash`` as the numpy-facing drop-in
(``paper_2110_00511_b200.numpy_api``): the map, set, heap and geometry names
resolve to the device implementation; every other reference submodule
(``tsdf``, ``bench``, ``io``, ``cli``, ``hashing``, ``backends``,
``serialize``, ``report``) is imported unmodified from the reference's own
sources, so e.g. ``spatialhash.tsdf.grid``'s ``from ..hashmap import
HashMap`` binds to the device map.  ``spatialhash_arrays`` (the reference's
array wrapper, which binds ``spatialhash`` as ``_native``) is likewise the
reference's own code running on the drop-in.

Environment: ``ASH_REF_PKG`` = directory holding the reference
``spatialhash`` package sources; ``ASH_REF_BINDINGS`` = directory holding
``spatialhash_arrays`` (both staged by tools/stage_reference_suite.sh).
"""
from __future__ import annotations

import os
import sys
import types
from pathlib import Path

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))

import paper_2110_00511_b200.numpy_api as _api  # noqa: E402

_pkg_dir = Path(os.environ["ASH_REF_PKG"]) / "spatialhash"
mod = types.ModuleType("spatialhash")
mod.__dict__.update({k: getattr(_api, k) for k in _api.__all__})
mod.__version__ = _api.__version__
mod.__path__ = [str(_pkg_dir)]  # reference submodules load from the reference sources
mod.__file__ = str(_pkg_dir / "__init__.py")
mod.__package__ = "spatialhash"
sys.modules["spatialhash"] = mod
for sub in ("hashmap", "index_heap", "geometry"):
    sys.modules[f"spatialhash.{sub}"] = _api
    setattr(mod, sub, _api)
if os.environ.get("ASH_REF_BINDINGS"):
    sys.path.insert(0, os.environ["ASH_REF_BINDINGS"])
