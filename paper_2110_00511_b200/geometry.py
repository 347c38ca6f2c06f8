"""Batch geometry on the device map: quantize and voxel_downsample.

Mirrors /root/reference/pkg/src/spatialhash/geometry.py:49-76.  Quantization
is float64 true division then floor (geometry.py:53), so float32 clouds are
widened exactly on the device and match the reference bit-for-bit.
voxel_downsample is one fused pass: quantize + set insert with the
first-occurrence winner + ascending select (libash ``ash_voxelize``).
"""
from __future__ import annotations

import os
import threading

import numpy as np
import torch

from . import _lib
from ._lib import AshMap, call
from .hashmap import BatchResult, HashMap, HashSet, _stream_handle, _table_slots

__all__ = ["PointCloud", "quantize", "voxel_downsample", "lattice_offsets", "radius_neighbors",
           "set_intersection", "cube_embed"]


class PointCloud:
    """Positions (float64, (n, 3)) plus optional per-point attributes
    (geometry.py:16-46).  Positions may be a CUDA tensor."""

    def __init__(self, positions, colors=None, normals=None):
        if isinstance(positions, torch.Tensor):
            self.positions = positions.to(torch.float64).reshape(-1, 3)
        else:
            self.positions = np.asarray(positions, dtype=np.float64).reshape(-1, 3)
        n = len(self.positions)
        for name, attr in (("colors", colors), ("normals", normals)):
            if attr is not None:
                attr = attr if isinstance(attr, torch.Tensor) else np.atleast_2d(np.asarray(attr))
                if attr.shape[0] != n:
                    attr = attr.reshape(n, -1)
                if attr.shape[0] != n:
                    raise ValueError(f"{name} length {attr.shape[0]} != {n} points")
            setattr(self, name, attr)

    def __len__(self) -> int:
        return len(self.positions)

    def select(self, idx) -> "PointCloud":
        if isinstance(self.positions, np.ndarray) and isinstance(idx, torch.Tensor):
            idx = idx.cpu().numpy()
        return PointCloud(self.positions[idx],
                          None if self.colors is None else self.colors[idx],
                          None if self.normals is None else self.normals[idx])


def _on_host(x) -> bool:
    """Results follow the input: host inputs (numpy, lists, CPU tensors)
    get host results, CUDA inputs get CUDA results."""
    pos = getattr(x, "positions", x)
    return not (isinstance(pos, torch.Tensor) and pos.is_cuda)


def _points_tensor(points, device) -> torch.Tensor:
    """(n, 3) float32/float64 on the device; other dtypes widen to float64
    (PointCloud stores float64, geometry.py:25)."""
    pos = getattr(points, "positions", points)
    if isinstance(pos, torch.Tensor):
        t = pos if pos.dtype in (torch.float32, torch.float64) else pos.to(torch.float64)
    else:
        a = np.asarray(pos)
        if a.dtype not in (np.float32, np.float64):
            a = a.astype(np.float64)
        t = torch.from_numpy(np.ascontiguousarray(a))
    t = t.reshape(-1, 3)
    return t.to(device, non_blocking=True).contiguous()


def _device(device) -> torch.device:
    dev = torch.device(device) if device is not None else \
        torch.device("cuda", torch.cuda.current_device())
    if dev.type == "cuda" and dev.index is None:
        dev = torch.device("cuda", torch.cuda.current_device())
    _lib.device_setup(dev)
    return dev


def quantize(positions, cell: float, device=None) -> torch.Tensor:
    """floor(p / cell) as int32 voxel coordinates (geometry.py:49-56)."""
    if cell <= 0:
        raise ValueError("cell size must be > 0")
    dev = _device(device)
    host = _on_host(positions)
    pts = _points_tensor(positions, dev)
    n = pts.shape[0]
    out = torch.empty((n, 3), dtype=torch.int32, device=dev)
    if n == 0:
        return out.cpu() if host else out
    flags = torch.zeros(1, dtype=torch.int32, device=dev)
    with torch.cuda.device(dev):
        call("ash_quantize", pts.data_ptr(), int(pts.dtype == torch.float64), n, float(cell),
             out.data_ptr(), flags.data_ptr(), _stream_handle(dev))
    if int(flags.item()) & _lib.FLAG_RANGE:
        raise ValueError("quantized coordinates exceed int32 range")
    return out.cpu() if host else out


class _VoxelWorkspace:
    """Per-device all-EMPTY table reused across voxelize calls; the select
    kernel restores every slot it claimed, so no per-call clear is needed.

    The table must hold every distinct voxel of a call.  2n slots always do,
    but the dedup is fastest when the table is small enough for its touched
    buckets to stay in the L2 (20M points at 5 mm: 702K voxels; a 40M-slot
    table spreads them over 640 MB).  A call is therefore tried on a prefix of
    ``4 x (voxels of the previous call)`` slots with a bounded probe; if that
    overflows (ASH_FLAG_TABLE_FULL) the prefix is refilled with EMPTY and the
    call repeats on the 2n-slot table (unbounded probe)."""

    _lock = threading.Lock()
    _by_device: dict = {}

    def __init__(self, device: torch.device):
        self.device = device
        self.slots = torch.empty(0, dtype=torch.int32, device=device)
        self.n_slots = 0
        self.counters = torch.zeros(_lib.N_COUNTERS, dtype=torch.int32, device=device)
        self.scan = torch.zeros(0, dtype=torch.int64, device=device)
        self.struct = AshMap()
        self.struct.arity = 3
        self.struct.counters = self.counters.data_ptr()
        self.estimate = 0  # distinct keys of the previous call
        self._seq_bufs = None
        self._reserved = -1  # batch size of the last reserve()

    @classmethod
    def get(cls, device: torch.device) -> "_VoxelWorkspace":
        with cls._lock:
            ws = cls._by_device.get(device)
            if ws is None:
                ws = cls._by_device[device] = cls(device)
            return ws

    SMALL_MIN = 1 << 16
    ESTIMATE_FACTOR = float(os.environ.get("ASH_WS_FACTOR", "4"))  # slots per distinct key of the previous call
    PROBE_LIMIT = 64  # buckets, for the estimated-size attempt

    def reserve(self, n: int) -> None:
        if n == self._reserved:  # the per-frame case: same batch size, nothing to size
            return
        need = _table_slots(max(n, 1), 2.0)
        if need > self.n_slots:
            self.slots = torch.empty(need * 4, dtype=torch.int32, device=self.device)
            self.n_slots = need
            call("ash_table_clear", self.slots.data_ptr(), need, _stream_handle(self.device))
            self.struct.slots = self.slots.data_ptr()
        self.full_slots = need
        tiles = _lib.scan_tiles(max(n, 1))
        if self.scan.numel() < tiles:
            self.scan = torch.zeros(tiles, dtype=torch.int64, device=self.device)
            self.struct.scan_status = self.scan.data_ptr()
            self.struct.scan_status_len = tiles
            self.tiles = torch.zeros(tiles, dtype=torch.int32, device=self.device)
            self.struct.tile_counts = self.tiles.data_ptr()
            self.struct.tile_counts_len = tiles
        self._reserved = n

    def sequence_buffers(self, n: int):
        """(blocks, gi, gmask, scratch_idx, scratch_mask, status) for a fused
        allocate of n candidates, reused while n repeats (stable pointers)."""
        if self._seq_bufs is None or self._seq_bufs[0] != n:
            dev = self.device
            self._seq_bufs = (n, torch.empty((n, 3), dtype=torch.int32, device=dev),
                              torch.empty(n, dtype=torch.int32, device=dev),
                              torch.empty(n, dtype=torch.uint8, device=dev),
                              torch.empty(n, dtype=torch.int32, device=dev),
                              torch.empty(8 * ((n + 31) // 32), dtype=torch.uint8, device=dev),  # cand / dem bitmaps
                              torch.empty(5, dtype=torch.int32, device=dev))
        return self._seq_bufs[1:]

    def attempts(self):
        """(table slots, probe limit) to try in order: the estimate-sized
        prefix first when it is smaller than the full table."""
        small = _table_slots(max(self.ESTIMATE_FACTOR * self.estimate, self.SMALL_MIN), 1.0)
        if self.estimate and small < self.full_slots:
            yield small, self.PROBE_LIMIT
        yield self.full_slots, 0

    def use(self, slots: int, max_probe: int) -> None:
        self.struct.n_slots = slots
        self.struct.max_probe = max_probe

    def refill(self, slots: int) -> None:
        call("ash_table_clear", self.slots.data_ptr(), slots, _stream_handle(self.device))

    def run(self, launch) -> tuple:
        """Run `launch()` (one fused dedup call) on the smallest table that
        holds the result; returns (count, flags) of the successful attempt."""
        for slots, probe in self.attempts():
            self.use(slots, probe)
            launch()
            # FLAGS (4) and COUNT (5) are adjacent: a view, one 8-byte read (no gather kernel)
            flags, count = self.counters[_lib.CTR_FLAGS:_lib.CTR_COUNT + 1].tolist()
            if probe and flags & _lib.FLAG_TABLE_FULL:
                self.refill(slots)  # claimed slots stay claimed after an overflow
                continue
            self.estimate = count
            return count, flags
        raise RuntimeError("voxel workspace overflow")  # unreachable: 2n slots hold n keys


def voxel_downsample(points, voxel_size: float, backend: str = "generic", threads: int = 1,
                     device=None):
    """One representative point per occupied voxel (geometry.py:59-76).

    Returns ``(voxel_coords int32 (k,3), selected int64 (k,))`` in
    first-occurrence (ascending point index) order, exactly the reference's
    ``coords[flatnonzero(HashSet.insert(coords).masks)]`` and index list.
    """
    if backend not in ("generic", "delegate", "integer_delegate"):
        raise ValueError(f"unknown backend {backend!r}")
    if voxel_size <= 0:
        raise ValueError("cell size must be > 0")
    dev = _device(device)
    host = _on_host(points)
    pts = _points_tensor(points, dev)
    n = pts.shape[0]
    if n == 0:
        z = (torch.zeros((0, 3), dtype=torch.int32), torch.zeros(0, dtype=torch.int64))
        return z if host else (z[0].to(dev), z[1].to(dev))
    ws = _VoxelWorkspace.get(dev)
    with _VoxelWorkspace._lock, torch.cuda.device(dev):
        ws.reserve(n)
        coords = torch.empty((n, 3), dtype=torch.int32, device=dev)
        sel = torch.empty(n, dtype=torch.int64, device=dev)
        scratch_idx = torch.empty(n, dtype=torch.int32, device=dev)
        scratch_mask = torch.empty(8 * ((n + 31) // 32), dtype=torch.uint8, device=dev)  # cand / dem bitmaps
        count, flags = ws.run(lambda: call(
            "ash_voxelize", _lib.ctypes.byref(ws.struct), pts.data_ptr(), int(pts.dtype == torch.float64), n,
            float(voxel_size), coords.data_ptr(), sel.data_ptr(), scratch_idx.data_ptr(),
            scratch_mask.data_ptr(), _stream_handle(dev)))
    if flags & _lib.FLAG_RANGE:
        raise ValueError("quantized coordinates exceed int32 range")
    if host:
        return coords[:count].cpu(), sel[:count].cpu()
    return coords[:count], sel[:count]


def lattice_offsets(r: int) -> torch.Tensor:
    """(2r+1)^3 offsets in [-r, r]^3, lexicographic (geometry.py:79-84)."""
    if r < 0:
        raise ValueError("radius must be >= 0")
    ax = torch.arange(-r, r + 1, dtype=torch.int32)
    g = torch.stack(torch.meshgrid(ax, ax, ax, indexing="ij"), dim=-1)
    return g.reshape(-1, 3)


def radius_neighbors(hashmap: HashMap, coords, r: int = 1) -> BatchResult:
    """find() of every lattice offset around each coordinate
    (geometry.py:87-99); results shaped (n, (2r+1)^3), column j is
    ``lattice_offsets(r)[j]``.  One kernel generates the offset queries on
    the fly (libash ``ash_find_lattice``); r = 0 is exactly ``find``."""
    if r < 0:
        raise ValueError("radius must be >= 0")
    host = HashMap._is_host(coords)
    if isinstance(coords, torch.Tensor):
        c = coords.reshape(-1, 3)
        if c.is_floating_point():  # np.asarray(coords, dtype=np.int32) truncates
            c = c.to(torch.int32)
    else:
        c = torch.from_numpy(np.ascontiguousarray(np.asarray(coords, dtype=np.int32).reshape(-1, 3)))
    c = hashmap._check_keys(c)
    n, k = c.shape[0], (2 * r + 1) ** 3
    idx = torch.empty((n, k), dtype=torch.int32, device=hashmap.device)
    msk = torch.empty((n, k), dtype=torch.uint8, device=hashmap.device)
    with hashmap._guard.reading(), torch.cuda.device(hashmap.device):
        if n:
            call("ash_find_lattice", hashmap._ptr(), c.data_ptr(), n, int(r), idx.data_ptr(),
                 msk.data_ptr(), hashmap._stream())
    out = BatchResult(idx, msk.view(torch.bool))
    return BatchResult(out.indices.cpu(), out.masks.cpu()) if host else out


def set_intersection(keys_a, keys_b, backend: str = "generic", threads: int = 1,
                     device=None) -> torch.Tensor:
    """Rows of keys_b present in keys_a, duplicates kept (geometry.py:129-143)."""
    dev = _device(device)
    host = HashMap._is_host(keys_b)
    a = torch.as_tensor(np.atleast_2d(np.asarray(keys_a, dtype=np.int32))) \
        if not isinstance(keys_a, torch.Tensor) else keys_a.to(torch.int32)
    b = torch.as_tensor(np.atleast_2d(np.asarray(keys_b, dtype=np.int32))) \
        if not isinstance(keys_b, torch.Tensor) else keys_b.to(torch.int32)
    a, b = a.to(dev), b.to(dev)
    if a.shape[0] == 0 or b.shape[0] == 0:
        return b[:0].cpu() if host else b[:0]
    if a.shape[1] != b.shape[1]:
        raise ValueError("key arity mismatch between the two sets")
    probe = HashSet(a.shape[0], a.shape[1], backend=backend, device=dev)
    probe.insert(a)
    out = b[probe.find(b).masks]
    return out.cpu() if host else out


_CUBE_CORNERS = torch.tensor([[i >> 2 & 1, i >> 1 & 1, i & 1] for i in range(8)], dtype=torch.int32)


def cube_embed(points, grid_spacing: float, device=None):
    """Enclosing-cell corners and trilinear weights per point
    (geometry.py:105-126): ``(corners int32 (n, 8, 3), weights float64
    (n, 8))``, corner j = floor(p / spacing) + the j-th ``(0,1)^3`` offset in
    lexicographic order.  Not on the map path: exported for the
    drop-in surface and computed with fp64 tensor ops in the reference's
    order (true division, floor, ``w = w_x * w_y * w_z`` left to right), so
    the weights are bit-identical to numpy's."""
    if grid_spacing <= 0:
        raise ValueError("grid spacing must be > 0")
    dev = _device(device)
    host = _on_host(points.positions if isinstance(points, PointCloud) else points)
    pts = _points_tensor(points, dev).to(torch.float64)  # np.asarray(..., float64)
    scaled = pts / grid_spacing
    base = torch.floor(scaled)
    frac = scaled - base
    if base.numel() and (float(base.min()) < -(2 ** 31) or float(base.max()) >= 2 ** 31):
        raise ValueError("grid coordinates exceed int32 range")
    off = _CUBE_CORNERS.to(dev)
    corners = base.to(torch.int32)[:, None, :] + off[None, :, :]
    axis_w = torch.where(off[None, :, :] == 1, frac[:, None, :], 1.0 - frac[:, None, :])
    weights = axis_w[..., 0] * axis_w[..., 1] * axis_w[..., 2]
    return (corners.cpu(), weights.cpu()) if host else (corners, weights)
