"""Voxel-block allocation on the device map (the map calls of
/root/reference/pkg/src/spatialhash/tsdf/grid.py:127-150, Alg. 2 of the
paper): a per-frame local map dedups candidate block coordinates, the
survivors are activated in the persistent global map, and each local entry
stores its block's global buffer index."""
from __future__ import annotations

import contextlib
import ctypes

import numpy as np
import torch

from . import _lib
from ._lib import call
from .hashmap import HashMap, ValueSpec, _get_device, _stream_handle

__all__ = ["allocate_blocks", "BlockGrid", "frame_candidates", "frame_blocks", "allocate_frame",
           "LocalBlockMap", "unique_rows"]


def unique_rows(keys: torch.Tensor) -> torch.Tensor:
    """Distinct int3 rows of a device batch in first-occurrence order — the
    survivors ``coords[local.activate(coords).masks]`` of tsdf/grid.py:140-142
    — in one fused dedup pass on the shared workspace table (libash
    ``ash_unique_rows``), no per-frame local map."""
    from .geometry import _VoxelWorkspace
    dev = keys.device
    n = keys.shape[0]
    if n == 0:
        return keys[:0]
    ws = _VoxelWorkspace.get(dev)
    with _VoxelWorkspace._lock, torch.cuda.device(dev):
        ws.reserve(n)
        out = torch.empty((n, 3), dtype=torch.int32, device=dev)
        scratch_idx = torch.empty(n, dtype=torch.int32, device=dev)
        scratch_mask = torch.empty(8 * ((n + 31) // 32), dtype=torch.uint8, device=dev)  # cand / dem bitmaps
        count, _ = ws.run(lambda: call(
            "ash_unique_rows", ctypes.byref(ws.struct), keys.data_ptr(), n, out.data_ptr(), None,
            scratch_idx.data_ptr(), scratch_mask.data_ptr(), _stream_handle(dev)))
    return out[:count]


def allocate_blocks(global_map: HashMap, coords, threads: int = 1):
    """grid.py:136-150 for a given candidate batch.

    Returns ``(gi, local_map)``: global indices of the frame's distinct blocks
    (first-occurrence order) and the local map (block -> global index).  The
    distinct blocks and the global activate run as one device sequence with
    a single host read (libash ``ash_allocate_blocks``); the local map —
    needed only by frame-scoped queries (tsdf/raycast.py:32-35) — is built on
    first use with the reference's indices (``LocalBlockMap``)."""
    if not (isinstance(coords, torch.Tensor) and coords.dtype == torch.int32 and coords.dim() == 2
            and coords.shape[1] == 3 and coords.device == global_map.device and coords.is_contiguous()):
        coords = global_map._check_keys(coords).contiguous()  # (a device int3 batch needs no checks)
    if coords.shape[0] == 0:
        return torch.zeros(0, dtype=torch.int32, device=global_map.device), None
    if global_map.key_arity != 3:
        raise ValueError("block coordinates must have key arity 3")
    n = coords.shape[0]
    if not _fused_ok(global_map):  # delegate semantics: the host-planned activate
        survivors = unique_rows(coords)
        gi, _ = global_map.activate(survivors)
        return gi, LocalBlockMap(survivors, gi, n, global_map.device)
    blocks, gi = _allocate_fused(
        global_map, n, lambda ws, out, gi_, gm_, si, sm, st, small, stream: call(
            "ash_allocate_blocks", global_map._ptr(), ctypes.byref(ws.struct), coords.data_ptr(), n,
            out.data_ptr(), gi_.data_ptr(), gm_.data_ptr(), si.data_ptr(), sm.data_ptr(), st.data_ptr(),
            small, stream))
    return gi, LocalBlockMap(blocks, gi, n, global_map.device)


_SMALL_ACTIVATE = 8192  # k_activate_small's batch limit (ash_map.cu kSmallMax)


def _fused_ok(gm: HashMap) -> bool:
    """The fused sequence activates with generic-backend semantics."""
    return gm.backend_name != "delegate"


def _allocate_fused(gm: HashMap, n: int, launch):
    """Dedup + global activate as one device sequence (ash_allocate_blocks /
    ash_allocate_frame): one host read of the 5-word status.  Falls back to
    the host-checked activate (growth, CapacityError) when the device guard
    reports that the new blocks did not fit.  Returns (blocks, gi)."""
    from .geometry import _VoxelWorkspace
    dev = gm.device
    ws = _VoxelWorkspace.get(dev)
    same_dev = _get_device is not None and torch.cuda.is_initialized() and dev.index == _get_device()
    with _VoxelWorkspace._lock, (contextlib.nullcontext() if same_dev else torch.cuda.device(dev)), \
            gm._guard.writing():
        gm._settle()
        ws.reserve(n)
        gm._ensure_scan(n)
        # the new blocks are at most capacity - size (else the device guard
        # rejects the batch): keep even that many claims under the slot limit
        gm._reserve_slots(max(gm._capacity - gm._top_ub, 0))
        # per-size buffers kept by the workspace: a repeated sequence keeps
        # its pointers and replays from libash's graph cache
        out, gi, gmask, scratch_idx, scratch_mask, status = ws.sequence_buffers(n)
        stream = _stream_handle(dev)
        for slots, probe in ws.attempts():
            ws.use(slots, probe)
            # one-block activate when the previous frame had few distinct blocks
            small = 1 if 2 * ws.estimate <= _SMALL_ACTIVATE else 0
            launch(ws, out, gi, gmask, scratch_idx, scratch_mask, status, small, stream)
            # the caller's result copies go in before the count is known
            # (sized from the previous call): no launch after the host read
            cap = min(n, max(256, 2 * ws.estimate))
            res = torch.empty(4 * cap, dtype=torch.int32, device=dev)  # one allocation for both
            blocks_c, gi_c = res[:3 * cap].view(cap, 3), res[3 * cap:]
            call("ash_copy_prefix2", out.data_ptr(), blocks_c.data_ptr(), 12, gi.data_ptr(), gi_c.data_ptr(), 4,
                 status.data_ptr() + 4, cap, stream)
            rows, count, wflags, gflags, winners = status.tolist()  # the one host read
            if probe and wflags & _lib.FLAG_TABLE_FULL:
                continue  # the workspace prefix overflowed (the global map was not touched)
            ws.estimate = count
            break
        else:  # unreachable: the full workspace table holds every distinct row
            raise RuntimeError("voxel workspace overflow")
        if wflags & _lib.FLAG_RANGE:
            raise ValueError("block coordinates exceed int32 range")
        gm._size_known = False
        if gflags & (_lib.FLAG_CAPACITY | _lib.FLAG_TABLE_FULL) or rows < count:
            # not committed on the device (more distinct blocks than the
            # capacity, or the guard fired): undo any claims, then the
            # host-checked activate (doubling growth, hashmap.py:389-396)
            if rows:
                call("ash_insert_rollback", gm._ptr(), rows, gi.data_ptr(), stream)
                gm._tombs_ub += rows
            blocks = out[:count].clone()
            return blocks, gm._insert_like(blocks, None, association=True).indices
        gm._top_ub = min(gm._capacity, gm._top_ub + winners)
        if count <= cap:
            return blocks_c[:count], gi_c[:count]
        return out[:count].clone(), gi[:count].clone()


class BlockGrid:
    """Global block map with dense (l, l, l, 2) float32 payloads
    (tsdf/grid.py:47-68); ``allocate(coords)`` runs the double-map scheme."""

    def __init__(self, block_resolution: int = 8, capacity: int = 10000,
                 with_color: bool = False, device=None, voxel_size: float = 0.0058,
                 trunc: float = 0.04, allocation: str = "ray"):
        if allocation not in ("ray", "neighbor"):
            raise ValueError("allocation must be 'ray' or 'neighbor'")
        l = int(block_resolution)
        self.voxel_size, self.trunc, self.allocation = float(voxel_size), float(trunc), allocation
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
    def block_size(self) -> float:
        """Block edge in meters (TsdfConfig.block_size, tsdf/types.py:102-104)."""
        return self.voxel_size * self.block_resolution

    def allocate_frame(self, depth, intrinsics, pose, depth_min: float = 0.2,
                       depth_max: float = 3.0) -> torch.Tensor:
        """VoxelBlockGrid.allocate_blocks(frame) (tsdf/grid.py:127-150) from
        the depth image, candidates generated on the device."""
        gi, local = allocate_frame(self.global_map, depth, intrinsics, pose, self.block_size,
                                   self.trunc, depth_min, depth_max, self.allocation)
        self.local_map = local
        self._local_indices = gi
        return gi

    @property
    def block_count(self) -> int:
        return self.global_map.size


# -- fused frame path (§8(f) row 1: tsdf/grid.py:98-150 from the depth image) --

def _frame_args(depth, intrinsics, pose, block_size: float, trunc: float, depth_min: float,
                depth_max: float, allocation: str, device):
    if allocation not in ("ray", "neighbor"):
        raise ValueError("allocation must be 'ray' or 'neighbor'")
    if not depth_min < depth_max:
        raise ValueError("depth_min must be < depth_max")
    if isinstance(depth, torch.Tensor):
        d = depth.to(device=device, dtype=torch.float64).contiguous()
    else:
        d = torch.from_numpy(np.ascontiguousarray(np.asarray(depth, dtype=np.float64))).to(device)
    if d.dim() != 2:
        raise ValueError("depth must be a (height, width) image")
    h, w = d.shape
    iw, ih = getattr(intrinsics, "width", w), getattr(intrinsics, "height", h)
    if (ih, iw) != (h, w):
        raise ValueError(f"depth shape {(h, w)} does not match intrinsics ({ih}, {iw})")
    cam = (ctypes.c_double * 6)(float(intrinsics.fx), float(intrinsics.fy), float(intrinsics.cx),
                                float(intrinsics.cy), float(depth_min), float(depth_max))
    p = np.asarray(pose, dtype=np.float64).reshape(4, 4)
    pose_c = (ctypes.c_double * 16)(*p.ravel().tolist())
    return d, h, w, cam, pose_c, int(allocation == "neighbor")


def frame_candidates(depth, intrinsics, pose, block_size: float, trunc: float,
                     depth_min: float = 0.2, depth_max: float = 3.0, allocation: str = "ray",
                     device=None) -> torch.Tensor:
    """The frame's block candidates in the reference's order
    (VoxelBlockGrid._candidate_blocks, tsdf/grid.py:98-125): valid pixels
    row-major, then ray samples (or the 27 lattice neighbours)."""
    from .geometry import _device
    dev = _device(device)
    d, h, w, cam, pose_c, nb = _frame_args(depth, intrinsics, pose, block_size, trunc, depth_min,
                                           depth_max, allocation, dev)
    n = int(_lib.lib.ash_frame_positions(h, w, float(block_size), float(trunc), nb))
    out = torch.empty((n, 3), dtype=torch.int32, device=dev)
    valid = torch.empty(n, dtype=torch.uint8, device=dev)
    flags = torch.zeros(1, dtype=torch.int32, device=dev)
    if n:
        with torch.cuda.device(dev):
            call("ash_frame_candidates", d.data_ptr(), h, w, cam, pose_c, float(block_size), float(trunc),
                 nb, out.data_ptr(), valid.data_ptr(), flags.data_ptr(), _stream_handle(dev))
    if int(flags.item()) & _lib.FLAG_RANGE:
        raise ValueError("block coordinates exceed int32 range")
    return out[valid.view(torch.bool)]


def frame_blocks(depth, intrinsics, pose, block_size: float, trunc: float,
                 depth_min: float = 0.2, depth_max: float = 3.0, allocation: str = "ray",
                 device=None) -> torch.Tensor:
    """Distinct block coordinates of the frame in first-occurrence order —
    ``coords[local.activate(coords).masks]`` of tsdf/grid.py:140-142 — in one
    fused pass (candidate generation + quantise + dedup, libash
    ``ash_frame_blocks``); the candidate list is never materialised."""
    from .geometry import _device, _VoxelWorkspace
    dev = _device(device)
    d, h, w, cam, pose_c, nb = _frame_args(depth, intrinsics, pose, block_size, trunc, depth_min,
                                           depth_max, allocation, dev)
    n = int(_lib.lib.ash_frame_positions(h, w, float(block_size), float(trunc), nb))
    if n == 0:
        return torch.zeros((0, 3), dtype=torch.int32, device=dev)
    ws = _VoxelWorkspace.get(dev)
    with _VoxelWorkspace._lock, torch.cuda.device(dev):
        ws.reserve(n)
        coords = torch.empty((n, 3), dtype=torch.int32, device=dev)
        scratch_idx = torch.empty(n, dtype=torch.int32, device=dev)
        scratch_mask = torch.empty(8 * ((n + 31) // 32), dtype=torch.uint8, device=dev)  # cand / dem bitmaps
        count, flags = ws.run(lambda: call(
            "ash_frame_blocks", ctypes.byref(ws.struct), d.data_ptr(), h, w, cam, pose_c, float(block_size),
            float(trunc), nb, coords.data_ptr(), scratch_idx.data_ptr(), scratch_mask.data_ptr(),
            _stream_handle(dev)))
    if flags & _lib.FLAG_RANGE:
        raise ValueError("block coordinates exceed int32 range")
    return coords[:count]


class LocalBlockMap:
    """The per-frame local map of tsdf/grid.py:140-149 (block coordinate ->
    global buffer index), built on first use from the frame's distinct blocks:
    activating them in first-occurrence order gives the same indices the
    reference's activate over the full candidate list gives (winner ranks)."""

    def __init__(self, blocks: torch.Tensor, gi: torch.Tensor, n_candidates, device):
        self._blocks, self._gi, self._n, self._device = blocks, gi, n_candidates, device
        self._map = None

    @property
    def map(self) -> HashMap:
        if self._map is None:
            n = self._n() if callable(self._n) else self._n  # capacity = len(candidates)
            m = HashMap(max(int(n), 1), 3, value_specs=[np.int32], device=self._device)
            li, _ = m.activate(self._blocks)
            m.value_buffer(0)[li.long(), 0] = self._gi
            self._map = m
        return self._map

    def __getattr__(self, name):
        return getattr(self.map, name)


def allocate_frame(global_map: HashMap, depth, intrinsics, pose, block_size: float, trunc: float,
                   depth_min: float = 0.2, depth_max: float = 3.0, allocation: str = "ray"):
    """VoxelBlockGrid.allocate_blocks (tsdf/grid.py:127-150) from the depth
    image: candidate generation, dedup and the global activate (whose
    indices are the frame's global buffer indices; the reference's follow-up
    find returns the same) as one device sequence with a single host read
    (libash ``ash_allocate_frame``).  Returns ``(gi, local_map)``."""
    dev = global_map.device
    if global_map.key_arity != 3:
        raise ValueError("block coordinates must have key arity 3")
    d, h, w, cam, pose_c, nb = _frame_args(depth, intrinsics, pose, block_size, trunc, depth_min,
                                           depth_max, allocation, dev)
    n = int(_lib.lib.ash_frame_positions(h, w, float(block_size), float(trunc), nb))
    if n == 0:
        return torch.zeros(0, dtype=torch.int32, device=dev), None
    if not _fused_ok(global_map):
        blocks = frame_blocks(depth, intrinsics, pose, block_size, trunc, depth_min, depth_max,
                              allocation, device=dev)
        gi = global_map.activate(blocks).indices if blocks.shape[0] else blocks[:0, 0]
    else:
        blocks, gi = _allocate_fused(
        global_map, n, lambda ws, out, gi_, gm_, si, sm, st, small, stream: call(
            "ash_allocate_frame", global_map._ptr(), ctypes.byref(ws.struct), d.data_ptr(), h, w, cam, pose_c,
                float(block_size), float(trunc), nb, out.data_ptr(), gi_.data_ptr(), gm_.data_ptr(),
                si.data_ptr(), sm.data_ptr(), st.data_ptr(), small, stream))
    if blocks.shape[0] == 0:
        return torch.zeros(0, dtype=torch.int32, device=dev), None
    per_pixel = n // (h * w)

    def n_candidates():  # valid pixels x samples (Frame.valid_mask, tsdf/types.py:67-69)
        valid = (d > 0) & (d >= depth_min) & (d <= depth_max)
        return int(valid.sum()) * per_pixel
    return gi, LocalBlockMap(blocks, gi, n_candidates, dev)
