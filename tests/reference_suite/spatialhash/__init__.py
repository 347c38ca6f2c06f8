"""``spatialhash`` shim: the reference's package name bound to the drop-in.

Put ``tests/reference_suite`` on PYTHONPATH (subprocesses inherit it, so
``python -m spatialhash.cli`` works too) and set ``ASH_REF_PKG`` to the
directory holding the reference ``spatialhash`` sources.  Then:

* ``spatialhash.{HashMap, HashSet, IndexHeap, voxel_downsample, ...}`` and
  the submodules ``spatialhash.hashmap`` / ``index_heap`` / ``geometry``
  are the numpy-facing drop-in (``paper_2110_00511_b200.numpy_api``; every
  batch op runs on the device through libash);
* every other submodule (``tsdf``, ``bench``, ``io``, ``cli``, ``hashing``,
  ``backends``, ``serialize``, ``report``) is imported unmodified from the
  reference sources, so e.g. ``spatialhash.tsdf.grid``'s
  ``from ..hashmap import HashMap`` binds to the device map.

Test infrastructure only (tests/test_reference_suite_gpu.py); the product
never imports it.
"""
import os
import sys
from pathlib import Path

_ROOT = Path(__file__).resolve().parents[3]
if str(_ROOT) not in sys.path:
    sys.path.insert(0, str(_ROOT))

import paper_2110_00511_b200.numpy_api as _api  # noqa: E402

globals().update({_k: getattr(_api, _k) for _k in _api.__all__})
__all__ = list(_api.__all__)
__version__ = _api.__version__
__path__.append(str(Path(os.environ["ASH_REF_PKG"]) / "spatialhash"))
for _sub in ("hashmap", "index_heap", "geometry"):
    sys.modules[f"{__name__}.{_sub}"] = _api
    globals()[_sub] = _api
