"""B200-native batch spatial hash map (ASH, arxiv 2110.00511).

Drop-in for the reference ``spatialhash`` package API
(/root/reference/pkg/src/spatialhash/__init__.py:3-16); every batch
operation runs hand-written sm_100a kernels from libash.so.

Names resolve lazily (PEP 562): importing the package, or a host-only
module such as ``workloads``, does not load libash.so; the first use of a
device name does, and raises if the library is missing (no CPU fallback).
"""
from __future__ import annotations

import importlib

__version__ = "0.1.0"

_EXPORTS = {
    "BatchResult": "hashmap", "CapacityError": "hashmap", "ConcurrentAccessError": "hashmap",
    "HashMap": "hashmap", "HashSet": "hashmap", "ValueSpec": "hashmap",
    "IndexHeap": "index_heap", "IndexHeapExhausted": "index_heap",
    "PointCloud": "geometry", "quantize": "geometry", "voxel_downsample": "geometry",
    "lattice_offsets": "geometry", "radius_neighbors": "geometry",
    "set_intersection": "geometry", "cube_embed": "geometry",
    "BlockGrid": "blocks", "allocate_blocks": "blocks", "allocate_frame": "blocks",
    "frame_blocks": "blocks", "frame_candidates": "blocks",
}

__all__ = sorted(_EXPORTS)


def __getattr__(name: str):
    mod = _EXPORTS.get(name)
    if mod is None:
        raise AttributeError(f"module {__name__!r} has no attribute {name!r}")
    value = getattr(importlib.import_module(f".{mod}", __name__), name)
    globals()[name] = value
    return value


def __dir__():
    return sorted(set(globals()) | set(_EXPORTS))
