"""B200-native batch spatial hash map (ASH, arxiv 2110.00511).

Drop-in for the reference ``spatialhash`` map API on CUDA tensors; every
batch operation runs hand-written sm_100a kernels from libash.so.
"""
from .hashmap import (BatchResult, CapacityError, ConcurrentAccessError, HashMap,
                      HashSet, ValueSpec)
from .geometry import (PointCloud, lattice_offsets, quantize, radius_neighbors,
                       set_intersection, voxel_downsample)
from .blocks import BlockGrid, allocate_blocks, allocate_frame, frame_blocks, frame_candidates

__version__ = "0.1.0"

__all__ = [
    "BatchResult", "CapacityError", "ConcurrentAccessError", "HashMap", "HashSet",
    "ValueSpec", "PointCloud", "quantize", "voxel_downsample", "lattice_offsets",
    "radius_neighbors", "set_intersection", "BlockGrid", "allocate_blocks",
    "allocate_frame", "frame_blocks", "frame_candidates",
]
