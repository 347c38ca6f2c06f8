"""numpy-facing form of the drop-in, for unmodified reference callers.

The reference ``spatialhash`` package takes and returns numpy arrays
(/root/reference/pkg/src/spatialhash/__init__.py:3-16); its consumers index
numpy arrays with ``BatchResult`` fields (tsdf/grid.py:140-147), call
``.copy()`` on buffer views and compare with numpy
(bindings/src/spatialhash_arrays/__init__.py:58-147).  The main package API
is torch-first (results follow the inputs; buffers are CUDA tensors).  This
module wraps the same device maps with numpy at the edges, so that

    import paper_2110_00511_b200.numpy_api as spatialhash

(or ``sys.modules["spatialhash"] = ...``) runs reference-shaped code as is.
Every operation still runs on the device through libash; only the host
conversions differ:

* batch results (``insert``/``activate``/``find``/``erase``,
  ``active_indices``, ``items_arrays``, geometry outputs) are numpy arrays;
* ``key_buffer`` is a read-only numpy snapshot of the device rows (item
  assignment raises ``ValueError`` as in hashmap.py:227-233);
* ``value_buffer(i)`` / ``value_buffers`` are numpy snapshots whose item
  assignment writes through to the device buffer (``buf[idx] = v`` and
  ``buf[idx, 0] += 1`` update the map, hashmap.py:235-242).  Deviation: a
  snapshot taken before a later batch does not see that batch's rows, and a
  basic-slice sub-view of a snapshot does not write through.
"""
from __future__ import annotations

import numpy as np
import torch

from . import geometry as _g
from . import hashmap as _h
from . import index_heap as _ih

__version__ = "0.1.0"

BatchResult = _h.BatchResult
CapacityError = _h.CapacityError
ConcurrentAccessError = _h.ConcurrentAccessError
ValueSpec = _h.ValueSpec
IndexHeapExhausted = _ih.IndexHeapExhausted

__all__ = [
    "BatchResult", "CapacityError", "ConcurrentAccessError", "HashMap",
    "HashSet", "IndexHeap", "IndexHeapExhausted", "PointCloud", "ValueSpec",
    "cube_embed", "lattice_offsets", "quantize", "radius_neighbors",
    "set_intersection", "voxel_downsample",
]


def _np(x):
    if isinstance(x, torch.Tensor):
        return x.detach().cpu().numpy()
    return x


def _result(r) -> BatchResult:
    return BatchResult(_np(r.indices), _np(r.masks))


def _torch_index(key, device):
    """A numpy-style index -> the equivalent torch index on ``device``."""
    if isinstance(key, tuple):
        return tuple(_torch_index(k, device) for k in key)
    if isinstance(key, (slice, int, type(None), type(Ellipsis))):
        return key
    if isinstance(key, np.integer):
        return int(key)
    if isinstance(key, torch.Tensor):
        return key.to(device)
    a = np.asarray(key)
    if a.dtype == np.bool_:
        return torch.from_numpy(np.ascontiguousarray(a)).to(device)
    return torch.from_numpy(np.ascontiguousarray(a.astype(np.int64))).to(device)


class DeviceRows(np.ndarray):
    """Host snapshot of a device value buffer; ``__setitem__`` writes the
    assigned region through to the device."""

    def __new__(cls, dev: torch.Tensor):
        obj = dev.detach().cpu().numpy().view(cls)
        obj._dev = dev
        return obj

    def __array_finalize__(self, obj):
        self._dev = None  # derived arrays (slices, results) are plain snapshots

    def __setitem__(self, key, value):
        np.ndarray.__setitem__(self, key, value)
        if self._dev is not None:
            region = np.ascontiguousarray(np.asarray(self.view(np.ndarray)[key]))
            self._dev[_torch_index(key, self._dev.device)] = torch.from_numpy(region).to(self._dev.device)

    def copy(self, order="C"):
        return np.array(self.view(np.ndarray), order=order, copy=True)


class HashMap(_h.HashMap):
    """``spatialhash.HashMap`` with numpy results (hashmap.py:153-515)."""

    def insert(self, keys, *values) -> BatchResult:
        return _result(super().insert(keys, *values))

    def activate(self, keys) -> BatchResult:
        return _result(super().activate(keys))

    def find(self, keys) -> BatchResult:
        return _result(super().find(keys))

    def erase(self, keys) -> np.ndarray:
        return _np(super().erase(keys))

    def active_indices(self) -> np.ndarray:
        return _np(super().active_indices())

    active_buf_indices = active_indices

    def items_arrays(self) -> tuple:
        return tuple(_np(a) for a in super().items_arrays())

    @property
    def key_buffer(self) -> np.ndarray:
        a = self._key_buf.detach().cpu().numpy()
        a.setflags(write=False)
        return a

    key_tensor = key_buffer

    @property
    def value_buffers(self) -> tuple:
        return tuple(DeviceRows(b) for b in self._value_bufs)

    def value_buffer(self, i: int = 0) -> np.ndarray:
        return DeviceRows(self._value_bufs[i])

    value_tensor = value_buffer

    @classmethod
    def load(cls, path, backend=None, threads=1, device=None):
        from .serialize import load_map
        m, meta = load_map(path, backend=backend, threads=threads, device=device)
        m.__class__ = HashSet if not m.value_specs else cls
        return m, meta


class HashSet(HashMap):
    """Keys only (hashmap.py:499-515)."""

    def __init__(self, capacity: int, key_arity: int, backend: str = "generic", threads: int = 1,
                 auto_rehash: bool = True, device=None):
        super().__init__(capacity, key_arity, (), backend=backend, threads=threads,
                         auto_rehash=auto_rehash, device=device)


class IndexHeap(_ih.IndexHeap):
    """``spatialhash.IndexHeap`` with numpy views (index_heap.py:14-55)."""

    @property
    def heap(self) -> np.ndarray:
        return _np(self._heap)

    def allocate(self, count: int) -> np.ndarray:
        return _np(super().allocate(count))

    def free_set(self) -> np.ndarray:
        return _np(super().free_set())


class PointCloud(_g.PointCloud):
    """numpy positions/attributes (geometry.py:16-46)."""

    def __init__(self, positions, colors=None, normals=None):
        super().__init__(_np(positions), _np(colors), _np(normals))

    def select(self, idx) -> "PointCloud":
        return PointCloud(self.positions[idx],
                          None if self.colors is None else self.colors[idx],
                          None if self.normals is None else self.normals[idx])


def quantize(positions, cell: float) -> np.ndarray:
    return _np(_g.quantize(_np(positions), cell))


def voxel_downsample(points, voxel_size: float, backend: str = "generic", threads: int = 1):
    coords, sel = _g.voxel_downsample(points, voxel_size, backend=backend, threads=threads)
    return _np(coords), _np(sel)


def lattice_offsets(r: int) -> np.ndarray:
    return _np(_g.lattice_offsets(r))


def radius_neighbors(hashmap, coords, r: int = 1) -> BatchResult:
    return _result(_g.radius_neighbors(hashmap, coords, r))


def cube_embed(points, grid_spacing: float):
    corners, weights = _g.cube_embed(points, grid_spacing)
    return _np(corners), _np(weights)


def set_intersection(keys_a, keys_b, backend: str = "generic", threads: int = 1) -> np.ndarray:
    return _np(_g.set_intersection(keys_a, keys_b, backend=backend, threads=threads))
