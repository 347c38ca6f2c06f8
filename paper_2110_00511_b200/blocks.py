"""Voxel-block allocation on the device map (the map calls of
/root/reference/pkg/src/spatialhash/tsdf/grid.py:127-150, Alg. 2 of the
paper): a per-frame local map dedups candidate block coordinates, the
survivors are activated in the persistent global map, and each local entry
stores its block's global buffer index."""
from __future__ import annotations

import numpy as np
import torch

from .hashmap import HashMap, ValueSpec

__all__ = ["allocate_blocks", "BlockGrid"]


def allocate_blocks(global_map: HashMap, coords, threads: int = 1):
    """grid.py:136-150 for a given candidate batch.

    Returns ``(gi, local_map)``: global indices of the frame's distinct blocks
    (first-occurrence order) and the local dedup map whose value buffer 0
    holds each block's global index."""
    coords = global_map._check_keys(coords)
    if coords.shape[0] == 0:
        return torch.zeros(0, dtype=torch.int32, device=global_map.device), None
    local = HashMap(coords.shape[0], 3, value_specs=[np.int32], threads=threads,
                    device=global_map.device)
    li, lmask = local.activate(coords)
    survivors = coords[lmask]
    global_map.activate(survivors)
    gi, gmask = global_map.find(survivors)
    local.value_buffer(0)[li[lmask].long(), 0] = gi
    return gi, local


class BlockGrid:
    """Global block map with dense (l, l, l, 2) float32 payloads
    (tsdf/grid.py:47-68); ``allocate(coords)`` runs the double-map scheme."""

    def __init__(self, block_resolution: int = 8, capacity: int = 10000,
                 with_color: bool = False, device=None):
        l = int(block_resolution)
        specs = [ValueSpec((l, l, l, 2), np.float32)]
        if with_color:
            specs.append(ValueSpec((l, l, l, 3), np.float32))
        self.block_resolution = l
        self.global_map = HashMap(capacity, 3, value_specs=specs, device=device)
        self.local_map = None
        self._local_indices = None

    def allocate(self, coords) -> torch.Tensor:
        gi, local = allocate_blocks(self.global_map, coords)
        self.local_map = local
        self._local_indices = gi
        return gi

    @property
    def block_count(self) -> int:
        return self.global_map.size
