"""Index-first spatial hash map on B200 — host side of the drop-in.

Mirrors the reference ``spatialhash.HashMap`` / ``HashSet`` API
(/root/reference/pkg/src/spatialhash/hashmap.py:33-515): same constructor,
same batch operations, same error types and messages, same generic-backend
index semantics.  Storage is CUDA memory owned by torch tensors; every batch
operation is a hand-written sm_100a kernel sequence behind the C ABI in
``include/ash.h`` (libash.so).  There is no CPU path.

Host policy kept from the reference:
  * validation (hashmap.py:246-286) and the reader/writer guard (:91-122);
  * growth by doubling and the re-plan after a rehash (:311-332, :389-396);
  * CapacityError leaves the map unchanged (:317-324).

Differences in mechanism (not in results):
  * ``size`` is tracked lazily: a mutating batch does not synchronise with the
    device unless the host cannot prove the batch fits (capacity - an upper
    bound on size >= batch length).  Reading ``size`` synchronises.
  * Results (indices int32, masks bool) live where the keys came from: CUDA
    keys give CUDA tensors, host keys give host tensors; large pinned host
    batches are pipelined (chunked H2D / kernels / D2H overlap).
  * ``threads`` is accepted and ignored (the device is the parallelism).
"""
from __future__ import annotations

import functools
import math
import os
import threading
from dataclasses import dataclass
from typing import Iterator, Sequence

import numpy as np
import torch

from . import _lib
from ._lib import AshMap, call

__all__ = ["HashMap", "HashSet", "ValueSpec", "BatchResult", "CapacityError",
           "ConcurrentAccessError"]


class CapacityError(RuntimeError):
    """Batch does not fit and automatic rehashing is disabled (hashmap.py:33)."""


class ConcurrentAccessError(RuntimeError):
    """A mutating batch overlapped another operation (hashmap.py:37)."""


def _np_dtype(dt) -> np.dtype:
    if isinstance(dt, torch.dtype):
        return torch.empty(0, dtype=dt).numpy().dtype
    return np.dtype(dt)


def _torch_dtype(dt: np.dtype) -> torch.dtype:
    return torch.from_numpy(np.empty(0, dtype=dt)).dtype


@dataclass(frozen=True)
class ValueSpec:
    """Shape and dtype of one value buffer entry (hashmap.py:41-70)."""

    shape: tuple
    dtype: np.dtype

    @classmethod
    def coerce(cls, spec) -> "ValueSpec":
        if isinstance(spec, ValueSpec):
            return spec
        if isinstance(spec, tuple) and len(spec) == 2 and isinstance(spec[0], (tuple, list)):
            return cls(tuple(int(s) for s in spec[0]), spec[1])
        return cls((1,), spec)

    def __post_init__(self):
        object.__setattr__(self, "shape", tuple(int(s) for s in self.shape))
        object.__setattr__(self, "dtype", _np_dtype(self.dtype))
        if any(s < 0 for s in self.shape):
            raise ValueError("value shape dimensions must be >= 0")

    @property
    def count(self) -> int:
        return int(np.prod(self.shape, dtype=np.int64)) if self.shape else 1

    @property
    def nbytes(self) -> int:
        return self.count * self.dtype.itemsize


@dataclass
class BatchResult:
    """Buffer indices (int32) and masks (bool), parallel to the batch
    (hashmap.py:73-88).  Where ``masks`` is False the index is -1."""

    indices: torch.Tensor
    masks: torch.Tensor

    def __iter__(self) -> Iterator[torch.Tensor]:
        return iter((self.indices, self.masks))

    def __len__(self) -> int:
        return len(self.indices)


class _AccessGuard:
    """N readers or one writer; violations raise (hashmap.py:91-122).
    ``reading()`` / ``writing()`` return plain context objects (a generator
    context manager costs ~2 us per batch call)."""

    def __init__(self):
        self._lock = threading.Lock()
        self._readers = 0
        self._writing = False
        self._r = _Reading(self)
        self._w = _Writing(self)

    def reading(self) -> "_Reading":
        return self._r

    def writing(self) -> "_Writing":
        return self._w


class _Reading:
    __slots__ = ("g",)

    def __init__(self, g: _AccessGuard):
        self.g = g

    def __enter__(self):
        g = self.g
        with g._lock:
            if g._writing:
                raise ConcurrentAccessError("read overlapped a mutating batch")
            g._readers += 1

    def __exit__(self, *exc):
        g = self.g
        with g._lock:
            g._readers -= 1
        return False


class _Writing:
    __slots__ = ("g",)

    def __init__(self, g: _AccessGuard):
        self.g = g

    def __enter__(self):
        g = self.g
        with g._lock:
            if g._writing or g._readers:
                raise ConcurrentAccessError("mutating batch requires exclusive map access")
            g._writing = True

    def __exit__(self, *exc):
        g = self.g
        with g._lock:
            g._writing = False
        return False


class ReadOnlyBuffer(torch.Tensor):
    """Tensor view whose item assignment and in-place ops raise ValueError,
    like the reference's non-writeable ``key_buffer`` (hashmap.py:227-233)."""

    def __setitem__(self, key, value):
        raise ValueError("assignment destination is read-only")

    @classmethod
    def __torch_function__(cls, func, types, args=(), kwargs=None):
        name = getattr(func, "__name__", "")
        inplace = (name.endswith("_") and not name.endswith("__")) or (
            name.startswith("__i") and name.endswith("__")
            and name not in ("__index__", "__int__", "__init__", "__iter__"))
        if inplace and args and isinstance(args[0], cls):
            raise ValueError("assignment destination is read-only")
        with torch._C.DisableTorchFunctionSubclass():
            return func(*args, **(kwargs or {}))


class _HeapView:
    """Read access matching ``IndexHeap`` (index_heap.py:14-55) for tests
    that inspect ``m._heap``."""

    def __init__(self, owner: "HashMap"):
        self._m = owner

    @property
    def capacity(self) -> int:
        return self._m.capacity

    @property
    def top(self) -> int:
        return self._m.size

    @property
    def free_count(self) -> int:
        return self._m.capacity - self._m.size

    @property
    def heap(self) -> torch.Tensor:
        return self._m._heap_buf

    def free_set(self) -> torch.Tensor:
        return self._m._heap_buf[self.top:].clone()


_raw_stream = getattr(torch._C, "_cuda_getCurrentRawStream", None)


def _stream_handle(device: torch.device) -> int:
    """The device's current stream as a raw handle (the C accessor skips
    torch.cuda.current_stream's device-index normalisation: ~2 us per call)."""
    if _raw_stream is not None and device.index is not None:
        return _raw_stream(device.index)
    return torch.cuda.current_stream(device).cuda_stream


_get_device = getattr(torch._C, "_cuda_getDevice", None)


def on_device(fn):
    """Run a map method with the map's GPU as the current device: libash
    launches on the calling thread's current device, and a stream handle of 0
    (a device's default stream) does not name one.  Already current: no
    device switch (the context costs ~3 us per call)."""
    @functools.wraps(fn)
    def wrapper(self, *args, **kwargs):
        idx = self._device.index
        if _get_device is not None and idx is not None and torch.cuda.is_initialized() and _get_device() == idx:
            return fn(self, *args, **kwargs)
        with torch.cuda.device(self._device):
            return fn(self, *args, **kwargs)
    return wrapper


# slots per unit of capacity (max live load 1/1.5); chosen by the r01 A/B
# matrix (tools/exp_matrix.sh): 1.5 beat 2.0 and 1.25 on the C2 sweep
TABLE_FACTOR = float(os.environ.get("ASH_TABLE_FACTOR", "1.5"))


def _table_slots(capacity: int, factor: float = None) -> int:
    """Even slot count = factor x capacity (live load factor <= 1/factor)."""
    f = TABLE_FACTOR if factor is None else factor
    n = max(64, int(math.ceil(capacity * f)))
    n += n & 1
    if n > 1 << 30:
        raise ValueError(f"capacity {capacity} exceeds the single-map table limit (2^30 slots)")
    return n


_SLOT_LIMIT = 0.75  # rebuild the table when non-EMPTY slots would pass this

# device insert batches run as sequential chunks of this many positions
# (0 = one batch); exact for insert, see HashMap._pipelined
INSERT_CHUNK = int(os.environ.get("ASH_INSERT_CHUNK", "0"))

# deferred slot-state commit (ash_insert_lazy / ash_settle): opt-in.  The
# sweep moves to the next mutating call, so it only saves work when a map is
# cleared or dropped before it is mutated again; finds meanwhile resolve
# PENDING slots through the rank words (~6% slower probes).  0 = eager sweep
LAZY_COMMIT = os.environ.get("ASH_LAZY_COMMIT", "0") == "1"


class HashMap:
    """Batch-parallel map from fixed-arity int32 keys to value buffers, on a
    CUDA device.  Signature of hashmap.py:178-196 plus ``device``."""

    def __init__(self, capacity: int, key_arity: int, value_specs: Sequence = (),
                 backend: str = "generic", threads: int = 1, auto_rehash: bool = True,
                 device=None):
        if capacity < 1:
            raise ValueError("capacity must be >= 1")
        if key_arity < 1:
            raise ValueError("key arity must be >= 1")
        if backend not in ("generic", "delegate", "integer_delegate"):
            raise ValueError(f"unknown backend {backend!r}")
        self.key_arity = int(key_arity)
        self.value_specs = tuple(ValueSpec.coerce(s) for s in value_specs)
        if len(self.value_specs) > _lib.MAX_VALUE_BUFFERS:
            raise ValueError(f"at most {_lib.MAX_VALUE_BUFFERS} value buffers are supported")
        self.backend_name = "delegate" if backend in ("delegate", "integer_delegate") else "generic"
        self.threads = max(1, int(threads))
        self.auto_rehash = bool(auto_rehash)
        self._device = torch.device(device) if device is not None else \
            torch.device("cuda", torch.cuda.current_device())
        if self._device.type != "cuda":
            raise ValueError("HashMap storage must be a CUDA device")
        if self._device.index is None:
            self._device = torch.device("cuda", torch.cuda.current_device())
        self._torch_dtypes = tuple(_torch_dtype(s.dtype) for s in self.value_specs)
        self._guard = _AccessGuard()
        self._debug_checksum = False
        self._heap = _HeapView(self)
        _lib.device_setup(self._device)
        self._init_state(int(capacity))

    # -- state ---------------------------------------------------------

    @on_device
    def _init_state(self, capacity: int, zero_rows: bool = True) -> None:
        """hashmap.py:200-210: fresh table, heap = arange, zeroed buffers.

        Everything is sized and allocated into locals first; the map's fields
        and the ctypes struct change only once all of it succeeded, so a
        rehash that fails (table limit ValueError, CUDA OOM) leaves the old
        map fully intact."""
        dev = self._device
        n_slots = _table_slots(capacity)  # raises past the table limit
        slots = torch.empty(n_slots * 4, dtype=torch.int32, device=dev)
        key_buf = torch.empty((capacity, self.key_arity), dtype=torch.int32, device=dev)
        value_bufs = tuple(torch.empty((capacity, *s.shape), dtype=td, device=dev)
                           for s, td in zip(self.value_specs, self._torch_dtypes))
        heap_buf = torch.empty(capacity, dtype=torch.int32, device=dev)
        active = torch.empty(capacity, dtype=torch.uint8, device=dev)
        erase_claim = torch.empty(capacity, dtype=torch.int32, device=dev)
        freed = torch.empty(capacity, dtype=torch.uint8, device=dev)
        counters = torch.zeros(_lib.N_COUNTERS, dtype=torch.int32, device=dev)
        need = _lib.scan_tiles(capacity)
        scan = torch.zeros(need, dtype=torch.int64, device=dev)
        tiles = torch.zeros(2 * need + 1, dtype=torch.int32, device=dev)
        rank_words = torch.empty(2 * (_lib.TILE // 32) * need, dtype=torch.int32, device=dev)
        # commit
        self._capacity = capacity
        self._n_slots = n_slots
        self._slots, self._key_buf, self._value_bufs = slots, key_buf, value_bufs
        self._heap_buf, self._active, self._erase_claim, self._freed = heap_buf, active, erase_claim, freed
        self._counters = counters
        self._scan, self._tiles, self._rank_words = scan, tiles, rank_words
        self._struct = AshMap()
        self._fill_struct()
        self._ensure_scan(capacity)
        call("ash_map_reset", self._ptr(), 1 if zero_rows else 0, self._stream())
        self._size = 0
        self._size_known = True
        self._top_ub = 0
        self._tombs_ub = 0
        self._unsettled = False

    def _settle(self) -> None:
        """Write the slot states a deferred commit left PENDING (libash
        ``ash_settle``: the table sweep of the last insert).  Every mutating
        operation calls it first; finds resolve pending slots on the fly, so
        an insert followed by finds and a clear() never pays the sweep."""
        if self._unsettled:
            call("ash_settle", self._ptr(), self._stream())
            self._unsettled = False

    def _fill_struct(self) -> None:
        s = self._struct
        s.slots = self._slots.data_ptr()
        s.n_slots = self._n_slots
        s.key_buf = self._key_buf.data_ptr()
        s.arity = self.key_arity
        s.n_values = len(self._value_bufs)
        for i, (buf, spec) in enumerate(zip(self._value_bufs, self.value_specs)):
            s.value_bufs[i] = buf.data_ptr()
            s.value_row_bytes[i] = spec.nbytes
        s.heap = self._heap_buf.data_ptr()
        s.active = self._active.data_ptr()
        s.erase_claim = self._erase_claim.data_ptr()
        s.freed = self._freed.data_ptr()
        s.counters = self._counters.data_ptr()
        s.capacity = self._capacity
        s.scan_status = self._scan.data_ptr()
        s.scan_status_len = self._scan.numel()
        s.tile_counts = self._tiles.data_ptr()
        s.tile_counts_len = self._tiles.numel()
        s.rank_words = self._rank_words.data_ptr()
        s.rank_words_len = self._rank_words.numel()

    def _ensure_scan(self, n: int) -> None:
        need = _lib.scan_tiles(max(n, self._capacity))
        if self._scan.numel() < need:
            # zeroed once; the library tags every launch with a fresh epoch
            self._scan = torch.zeros(max(need, 2 * self._scan.numel()), dtype=torch.int64,
                                     device=self._device)
            self._struct.scan_status = self._scan.data_ptr()
            self._struct.scan_status_len = self._scan.numel()
            # per-tile winner counts: zero between batches (the commit or the
            # rollback clears what the claim counted)
            # [0, T): counts, [T, 2T]: exclusive prefixes of the staged commit
            self._tiles = torch.zeros(2 * self._scan.numel() + 1, dtype=torch.int32,
                                      device=self._device)
            self._struct.tile_counts = self._tiles.data_ptr()
            self._struct.tile_counts_len = self._tiles.numel()
            # per 32 positions: winner bits + rank of the first (table-sweep commit)
            self._rank_words = torch.empty(2 * (_lib.TILE // 32) * self._scan.numel(),
                                           dtype=torch.int32, device=self._device)
            self._struct.rank_words = self._rank_words.data_ptr()
            self._struct.rank_words_len = self._rank_words.numel()


    def _ptr(self):
        return _lib.ctypes.byref(self._struct)

    def _stream(self) -> int:
        return _stream_handle(self._device)

    def _sync_size(self) -> int:
        if not self._size_known:
            self._size = int(self._counters[_lib.CTR_TOP].item())
            self._size_known = True
            self._top_ub = self._size
        return self._size

    @property
    def device(self) -> torch.device:
        return self._device

    @property
    def capacity(self) -> int:
        return self._capacity

    @property
    def bucket_count(self) -> int:
        """The reference's bucket count: capacity (generic) or 2x capacity
        (delegate), backends.py:187,233."""
        return self._capacity * (2 if self.backend_name == "delegate" else 1)

    @property
    def slot_count(self) -> int:
        """Open-addressing slots actually allocated on the device."""
        return self._n_slots

    @property
    def size(self) -> int:
        return self._sync_size()

    def __len__(self) -> int:
        return self._sync_size()

    @property
    def key_buffer(self) -> torch.Tensor:
        """Read-only (capacity, arity) int32 view (hashmap.py:227-233)."""
        return torch.Tensor._make_subclass(ReadOnlyBuffer, self._key_buf, False)

    @property
    def value_buffers(self) -> tuple:
        """Writable value buffers (hashmap.py:235-239)."""
        return self._value_bufs

    def value_buffer(self, i: int = 0) -> torch.Tensor:
        return self._value_bufs[i]

    # Open3D-style names used by north_star
    @property
    def key_tensor(self) -> torch.Tensor:
        return self.key_buffer

    def value_tensor(self, i: int = 0) -> torch.Tensor:
        return self.value_buffer(i)

    def active_buf_indices(self) -> torch.Tensor:
        return self.active_indices()

    @on_device
    def reserve(self, capacity: int) -> None:
        """Grow to at least ``capacity`` (no-op when already large enough)."""
        if int(capacity) > self._capacity:
            self.rehash(int(capacity))

    # -- validation (hashmap.py:246-286) --------------------------------

    def _check_keys(self, keys, to_device: bool = True) -> torch.Tensor:
        if (to_device and isinstance(keys, torch.Tensor) and keys.dtype == torch.int32 and keys.dim() == 2
                and keys.shape[1] == self.key_arity and keys.device == self._device and keys.is_contiguous()):
            return keys  # already a device int32 batch of this arity: nothing to check or move
        if isinstance(keys, torch.Tensor):
            k = keys
            if k.is_floating_point() or k.is_complex():
                raise ValueError("floating-point keys are not accepted; quantize to int32 first")
        else:
            arr = np.asarray(keys)
            if arr.dtype.kind == "f":
                raise ValueError("floating-point keys are not accepted; quantize to int32 first")
            if arr.dtype.kind not in "iub" and arr.size:
                raise ValueError(f"keys must be integers, got {arr.dtype}")
            if arr.size == 0 and arr.dtype.kind not in "iub":
                arr = arr.astype(np.int32)
            if arr.dtype != np.int32:
                cast = arr.astype(np.int32)
                if np.any(cast != arr):
                    raise ValueError("key values do not fit in int32")
                arr = cast
            k = torch.from_numpy(np.ascontiguousarray(arr))
        if k.dim() == 1:
            if self.key_arity == 1:
                k = k.reshape(-1, 1)
            elif k.numel() == self.key_arity:
                k = k.reshape(1, -1)
        if k.dim() != 2 or k.shape[1] != self.key_arity:
            raise ValueError(f"keys must have shape (n, {self.key_arity}), got {tuple(k.shape)}")
        if k.dtype != torch.int32:
            cast = k.to(torch.int32)
            if bool((cast.to(k.dtype) != k).any()):
                raise ValueError("key values do not fit in int32")
            k = cast
        return k.to(self._device, non_blocking=True).contiguous() if to_device else k.contiguous()

    def _check_values(self, m: int, values, to_device: bool = True) -> list:
        if len(values) != len(self.value_specs):
            raise ValueError(f"expected {len(self.value_specs)} value batches, got {len(values)}")
        out = []
        for pos, (spec, td, batch) in enumerate(zip(self.value_specs, self._torch_dtypes, values)):
            if isinstance(batch, torch.Tensor):
                t = batch.to(dtype=td)
            else:
                a = np.asarray(batch)
                if a.dtype != spec.dtype:
                    a = a.astype(spec.dtype)
                t = torch.from_numpy(np.ascontiguousarray(a))
            if t.dim() == 0 or (t.shape[0] != m and not (m == 0 and t.numel() == 0)):
                length = t.shape[0] if t.dim() else 1
                raise ValueError(f"value batch {pos} has length {length}, expected {m}")
            try:
                t = t.reshape((m, *spec.shape))
            except RuntimeError:
                raise ValueError(
                    f"value batch {pos} has shape {tuple(t.shape)}, expected "
                    f"(n, {', '.join(map(str, spec.shape))})") from None
            out.append(t.to(self._device, non_blocking=True).contiguous() if to_device else t.contiguous())
        return out

    # -- growth (hashmap.py:311-332) --------------------------------------

    def _grown_capacity(self, extra: int) -> int:
        size = self._sync_size()
        cap = self._capacity
        while cap - size < extra:
            cap *= 2
        return cap

    def _rehash_into(self, new_capacity: int) -> None:
        """Rebuild: active rows in ascending index order become rows
        0..size-1 of fresh zeroed buffers (hashmap.py:326-332)."""
        self._settle()
        size = self._sync_size()
        act = torch.empty(size, dtype=torch.int32, device=self._device)
        if size:
            call("ash_active_indices", self._ptr(), act.data_ptr(), self._stream())
        old = AshMap.from_buffer_copy(self._struct)
        keep = (self._slots, self._key_buf, self._value_bufs, self._heap_buf, self._active,
                self._erase_claim, self._freed, self._counters)
        self._init_state(new_capacity)
        if size:
            call("ash_rehash_from", self._ptr(), _lib.ctypes.byref(old), act.data_ptr(), size,
                 self._stream())
        del keep  # stream-ordered frees: the allocator reuses them only after these kernels
        self._size = size
        self._size_known = True
        self._top_ub = size
        self._tombs_ub = 0

    def _reserve_slots(self, m: int) -> None:
        """Keep non-EMPTY slots (live + tombstones + this batch's claims)
        under the probe limit; rebuilds the table in place (same indices)
        when erases left too many tombstones."""
        limit = int(_SLOT_LIMIT * self._n_slots)
        if self._top_ub + self._tombs_ub + m <= limit:
            return
        self._settle()
        tombs = int(self._counters[_lib.CTR_TOMBS].item())
        size = self._sync_size()
        self._tombs_ub = tombs
        if size + tombs + min(m, self._capacity - size) <= limit:
            return
        self._rebuild_slots(self._n_slots)

    def _rebuild_slots(self, n_slots: int) -> None:
        """Re-place every live slot into a fresh array of n_slots slots (same
        buffer indices; tombstones dropped)."""
        self._settle()
        new_slots = torch.empty(n_slots * 4, dtype=torch.int32, device=self._device)
        call("ash_rebuild_table", self._ptr(), new_slots.data_ptr(), n_slots, self._stream())
        self._slots = new_slots
        self._n_slots = n_slots
        self._struct.slots = new_slots.data_ptr()
        self._struct.n_slots = n_slots
        self._tombs_ub = 0

    def _widen_for_claims(self, m: int) -> None:
        """A batch longer than the free space claims up to m new slots
        before its exact winner count is known.  Make the slot array hold
        size + m under the load limit first (capacity and indices unchanged),
        so an oversize batch of distinct keys cannot run the table full and
        probe it end to end; the rehash that follows, if the winners do not
        fit, sizes the table from the new capacity again."""
        size = self._sync_size()
        tombs = int(self._counters[_lib.CTR_TOMBS].item())
        if size + tombs + m <= int(_SLOT_LIMIT * self._n_slots):
            return
        want = int(math.ceil((size + m) / _SLOT_LIMIT)) + 2
        want = min(1 << 30, max(self._n_slots, want + (want & 1)))
        self._rebuild_slots(want)

    # -- operations (hashmap.py:336-456) ---------------------------------

    # -- host-resident batches ---------------------------------------------
    # Results live where the keys came from: CUDA keys -> CUDA results; host
    # keys (numpy, lists, CPU tensors) -> host results, like the reference.
    # Large pinned host batches are pipelined in chunks: H2D of chunk i+1
    # overlaps the kernels of chunk i and the D2H of chunk i-1.  For insert
    # this is exact: a later position never demotes an earlier one, so a
    # chunk's winners are final after its own claim, and sequential chunks
    # give the single-batch masks and indices (found-earlier == duplicate
    # loser in insert mode: both report False / -1).

    PIPELINE_MIN = 1 << 20
    PIPELINE_CHUNK = int(os.environ.get("ASH_PIPELINE_CHUNK", 1 << 20))

    @staticmethod
    def _is_host(x) -> bool:
        return not (isinstance(x, torch.Tensor) and x.is_cuda)

    def _streams(self):
        if getattr(self, "_xfer", None) is None:
            self._xfer = (torch.cuda.Stream(self._device), torch.cuda.Stream(self._device))
        return self._xfer

    def _to_host(self, res: BatchResult) -> BatchResult:
        return BatchResult(res.indices.cpu(), res.masks.cpu())

    def _pipelined(self, keys_h: torch.Tensor, vals_h, op: str) -> BatchResult:
        """Chunked H2D / kernels / D2H overlap for a host batch (op = insert
        or find).  Caller holds the guard and has checked capacity."""
        if op == "insert":
            self._settle()
        m = keys_h.shape[0]
        dev = self._device
        s = torch.cuda.current_stream(dev)
        h2d, d2h = self._streams()
        keys_d = torch.empty((m, self.key_arity), dtype=torch.int32, device=dev)
        vals_d = [torch.empty((m, *v.shape[1:]), dtype=v.dtype, device=dev) for v in vals_h]
        idx_d = torch.empty(m, dtype=torch.int32, device=dev)
        msk_d = torch.empty(m, dtype=torch.uint8, device=dev)
        idx_h = torch.empty(m, dtype=torch.int32, pin_memory=True)
        msk_h = torch.empty(m, dtype=torch.uint8, pin_memory=True)
        h2d.wait_stream(s)
        d2h.wait_stream(s)
        c = self.PIPELINE_CHUNK
        self._ensure_scan(min(m, c))
        for a in range(0, m, c):
            b = min(m, a + c)
            with torch.cuda.stream(h2d):
                keys_d[a:b].copy_(keys_h[a:b], non_blocking=True)
                for vd, vh in zip(vals_d, vals_h):
                    vd[a:b].copy_(vh[a:b], non_blocking=True)
            s.wait_stream(h2d)
            if op == "insert":
                vptr = None
                if vals_d:
                    vptr = (_lib.c_void_p * len(vals_d))(*[v[a:b].data_ptr() for v in vals_d])
                call("ash_insert", self._ptr(), keys_d[a:b].data_ptr(), b - a, vptr, 0,
                     idx_d[a:b].data_ptr(), msk_d[a:b].data_ptr(), self._stream())
            else:
                call("ash_find", self._ptr(), keys_d[a:b].data_ptr(), b - a, idx_d[a:b].data_ptr(),
                     msk_d[a:b].data_ptr(), self._stream())
            d2h.wait_stream(s)
            with torch.cuda.stream(d2h):
                idx_h[a:b].copy_(idx_d[a:b], non_blocking=True)
                msk_h[a:b].copy_(msk_d[a:b], non_blocking=True)
        d2h.synchronize()
        return BatchResult(idx_h, msk_h.view(torch.bool))

    def _pipeline_fits(self, keys) -> bool:
        return (isinstance(keys, torch.Tensor) and not keys.is_cuda and keys.is_pinned()
                and keys.dim() == 2 and keys.shape[0] >= self.PIPELINE_MIN)

    @on_device
    def insert(self, keys, *values) -> BatchResult:
        """Insert keys with one value batch per value buffer: the first
        occurrence of each absent key wins a fresh index; existing values are
        never overwritten (hashmap.py:336-347)."""
        host = self._is_host(keys)
        if host and self._pipeline_fits(keys) and self.backend_name != "delegate":
            k = self._check_keys(keys, to_device=False)
            vals = self._check_values(k.shape[0], values, to_device=False)
            with self._guard.writing():
                m = k.shape[0]
                if m > self._capacity - self._top_ub:
                    self._sync_size()
                if m <= self._capacity - self._top_ub:
                    self._reserve_slots(m)
                    res = self._pipelined(k, vals, "insert")
                    self._top_ub = min(self._capacity, self._top_ub + m)
                    self._size_known = False
                    return res
                return self._to_host(self._insert_like(
                    k.to(self._device), [v.to(self._device) for v in vals], association=False))
        keys = self._check_keys(keys)
        vals = self._check_values(keys.shape[0], values)
        with self._guard.writing():
            res = self._insert_like(keys, vals, association=False)
        return self._to_host(res) if host else res

    @on_device
    def activate(self, keys) -> BatchResult:
        """Ensure keys are present; values untouched; masks = found OR
        winner (hashmap.py:349-360)."""
        host = self._is_host(keys)
        keys = self._check_keys(keys)
        with self._guard.writing():
            res = self._insert_like(keys, None, association=True)
        return self._to_host(res) if host else res

    def _insert_like(self, keys: torch.Tensor, vals, association: bool, idx=None) -> BatchResult:
        m = keys.shape[0]
        dev = self._device
        self._settle()
        if idx is None:
            idx = torch.empty(m, dtype=torch.int32, device=dev)
        msk = torch.empty(m, dtype=torch.uint8, device=dev)
        if m == 0:
            return BatchResult(idx, msk.view(torch.bool))
        vptr = None
        if vals is not None and len(vals):
            vptr = (_lib.c_void_p * len(vals))(*[v.data_ptr() for v in vals])
        assoc = 1 if association else 0
        if self.backend_name == "delegate":
            self._insert_delegate(keys, m, vptr, assoc, idx, msk)
            self._size_known = False
            return BatchResult(idx, msk.view(torch.bool))
        while True:
            self._reserve_slots(m)
            self._ensure_scan(m)
            if m > self._capacity - self._top_ub:
                self._sync_size()
            free = self._capacity - self._top_ub
            if m <= free:
                # the whole batch fits: fused path, no host synchronisation.
                # insert (not activate) may run as sequential chunks with
                # identical results (see _pipelined); a chunk's table lines
                # then stay L2-resident between its claim and its commit.
                c = INSERT_CHUNK if (not association and INSERT_CHUNK > 0) else m
                if c >= m:  # one call on the whole batch (no slicing)
                    call("ash_insert_lazy" if LAZY_COMMIT else "ash_insert", self._ptr(), keys.data_ptr(), m,
                         vptr, assoc, idx.data_ptr(), msk.data_ptr(), self._stream())
                    self._unsettled = LAZY_COMMIT
                chunks = range(0, m, c) if c < m else ()
                for a in chunks:
                    b = min(m, a + c)
                    cp = vptr
                    if vals:
                        cp = (_lib.c_void_p * len(vals))(*[v[a:b].data_ptr() for v in vals])
                    if c < m:
                        self._settle()  # a chunk's claim must see the previous chunk committed
                    call("ash_insert_lazy" if LAZY_COMMIT else "ash_insert", self._ptr(),
                         keys[a:b].data_ptr(), b - a, cp, assoc, idx[a:b].data_ptr(), msk[a:b].data_ptr(),
                         self._stream())
                    self._unsettled = LAZY_COMMIT
                self._top_ub = min(self._capacity, self._top_ub + m)
                break
            self._widen_for_claims(m)
            call("ash_insert_claim", self._ptr(), keys.data_ptr(), m, idx.data_ptr(),
                 msk.data_ptr(), self._stream())
            call("ash_insert_count", self._ptr(), m, idx.data_ptr(), msk.data_ptr(),
                 self._stream())
            winners = int(self._counters[_lib.CTR_WINNERS].item())
            if winners <= free:
                call("ash_insert_commit_lazy" if LAZY_COMMIT else "ash_insert_commit", self._ptr(),
                     keys.data_ptr(), m, vptr, assoc,
                     idx.data_ptr(), msk.data_ptr(), self._stream())
                self._unsettled = LAZY_COMMIT
                self._top_ub = min(self._capacity, self._top_ub + winners)
                break
            call("ash_insert_rollback", self._ptr(), m, idx.data_ptr(), self._stream())
            self._tombs_ub += m
            if not self.auto_rehash:
                raise CapacityError(
                    f"batch needs {winners} free slots, {free} available at capacity "
                    f"{self._capacity}")
            # rehash moves every slot, so plan again afterwards (hashmap.py:393-396)
            self._rehash_into(self._grown_capacity(winners))
        self._size_known = False
        return BatchResult(idx, msk.view(torch.bool))

    def _insert_delegate(self, keys, m, vptr, assoc, idx, msk) -> None:
        """Delegate backend (hashmap.py:369-387): the buffer must hold size + m
        during the call (growth is planned on m, not on the winners); position
        p owns heap[top + p]; losers return to the heap sorted with stale key
        rows (libash ash_insert_commit_delegate + ash_heap_put_losers)."""
        while True:
            self._reserve_slots(m)
            self._ensure_scan(m)
            if m > self._capacity - self._top_ub:
                self._sync_size()
            free = self._capacity - self._top_ub
            if m <= free:
                break
            if not self.auto_rehash:
                raise CapacityError(f"batch needs {m} free slots, {free} available at capacity "
                                    f"{self._capacity}")
            self._rehash_into(self._grown_capacity(m))
        losers = torch.full((m,), 2**31 - 1, dtype=torch.int32, device=self._device)
        call("ash_insert_claim", self._ptr(), keys.data_ptr(), m, idx.data_ptr(), msk.data_ptr(),
             self._stream())
        call("ash_insert_count", self._ptr(), m, idx.data_ptr(), msk.data_ptr(), self._stream())
        call("ash_insert_commit_delegate", self._ptr(), keys.data_ptr(), m, vptr, assoc,
             idx.data_ptr(), msk.data_ptr(), losers.data_ptr(), self._stream())
        srt = torch.sort(losers).values  # the sorted free of index_heap.py:46
        call("ash_heap_put_losers", self._ptr(), srt.data_ptr(), m, self._stream())
        self._top_ub = min(self._capacity, self._top_ub + m)

    @on_device
    def _op_into(self, op: str, keys: torch.Tensor, vals, out_idx: torch.Tensor) -> None:
        """insert / activate / find of a CUDA batch (already checked) with the
        indices written straight into out_idx, e.g. a view of the peer
        transport's result buffer (no copy); masks are derived by the caller
        (index >= 0)."""
        m = keys.shape[0]
        if op == "find":
            with self._guard.reading():
                if m:
                    msk = torch.empty(m, dtype=torch.uint8, device=self._device)
                    call("ash_find", self._ptr(), keys.data_ptr(), m, out_idx.data_ptr(),
                         msk.data_ptr(), self._stream())
            return
        if op not in ("insert", "activate"):
            raise ValueError(f"unknown op {op!r}")
        with self._guard.writing():
            self._insert_like(keys, vals if op == "insert" else None, op == "activate", idx=out_idx)

    def _dn_ready(self, op: str, n_max: int) -> bool:
        """Can a device-sized batch of up to n_max keys run with no host
        check?  find: always.  insert / activate: the generic backend with
        free indices and slots for all n_max (so the device capacity guard
        cannot fire)."""
        if op == "find":
            return True
        if self.backend_name == "delegate" or self._capacity - self._top_ub < n_max:
            return False
        return self._top_ub + self._tombs_ub + n_max <= int(_SLOT_LIMIT * self._n_slots)

    def _op_into_dn(self, op: str, keys: torch.Tensor, vals, out_idx: torch.Tensor, d_n: torch.Tensor) -> None:
        """insert / activate / find of keys[0 : d_n[0]) (device length, at most
        keys.shape[0]) with the indices written into out_idx (ash_insert_dn /
        ash_find_dn); the caller checked _dn_ready."""
        n_max = keys.shape[0]
        if not n_max:
            return
        msk = getattr(self, "_dn_mask", None)
        if msk is None or msk.numel() < n_max:
            msk = self._dn_mask = torch.empty(n_max, dtype=torch.uint8, device=self._device)
        if op == "find":
            with self._guard.reading():
                call("ash_find_dn", self._ptr(), keys.data_ptr(), n_max, d_n.data_ptr(), out_idx.data_ptr(),
                     msk.data_ptr(), self._stream())
            return
        with self._guard.writing():
            self._settle()
            self._ensure_scan(n_max)
            vptr = None
            if vals:
                vptr = (_lib.c_void_p * len(vals))(*[v.data_ptr() for v in vals])
            call("ash_insert_dn", self._ptr(), keys.data_ptr(), n_max, d_n.data_ptr(), vptr,
                 1 if op == "activate" else 0, out_idx.data_ptr(), msk.data_ptr(), self._stream())
            self._top_ub = min(self._capacity, self._top_ub + n_max)
            self._size_known = False

    def _dn_done(self, op: str) -> None:
        """After a device-sized insert: it can only fail on a probe chain past
        the device bound (load <= 0.75: not in practice).  The flags word is
        copied to pinned memory behind the op and checked at the next call
        (``_dn_check``), so the op itself never waits; a failure is raised
        loudly rather than returning wrong indices silently."""
        if op == "find":
            return
        if getattr(self, "_dn_flags_h", None) is None:
            self._dn_flags_h = torch.zeros(1, dtype=torch.int32, pin_memory=True)
            self._dn_flags_ev = torch.cuda.Event()
        self._dn_check()  # the previous one's flags (long arrived: one op back)
        self._dn_flags_h.copy_(self._counters[_lib.CTR_FLAGS:_lib.CTR_FLAGS + 1], non_blocking=True)
        self._dn_flags_ev.record(torch.cuda.current_stream(self._device))
        self._dn_pending = True

    def _dn_check(self, wait: bool = True) -> None:
        """Raise if a previous device-sized insert failed; wait=False only
        looks when its flags have already arrived (never blocks)."""
        if getattr(self, "_dn_pending", False):
            if not wait and not self._dn_flags_ev.query():
                return
            self._dn_flags_ev.synchronize()
            self._dn_pending = False
            if int(self._dn_flags_h[0]) & (_lib.FLAG_CAPACITY | _lib.FLAG_TABLE_FULL):
                raise RuntimeError("a device-sized insert could not place every key (probe bound); "
                                   "rebuild the map")

    @on_device
    def find(self, keys) -> BatchResult:
        """Look up keys; the map is not modified (hashmap.py:415-429)."""
        host = self._is_host(keys)
        if host and self._pipeline_fits(keys):
            k = self._check_keys(keys, to_device=False)
            with self._guard.reading():
                return self._pipelined(k, [], "find")
        keys = self._check_keys(keys)
        with self._guard.reading():
            m = keys.shape[0]
            idx = torch.empty(m, dtype=torch.int32, device=self._device)
            msk = torch.empty(m, dtype=torch.uint8, device=self._device)
            if m:
                call("ash_find", self._ptr(), keys.data_ptr(), m, idx.data_ptr(),
                     msk.data_ptr(), self._stream())
            res = BatchResult(idx, msk.view(torch.bool))
        return self._to_host(res) if host else res

    @on_device
    def erase(self, keys) -> torch.Tensor:
        """Remove keys; exactly one True per removed key, at its first batch
        position (hashmap.py:431-456)."""
        host = self._is_host(keys)
        keys = self._check_keys(keys)
        with self._guard.writing():
            m = keys.shape[0]
            out = torch.empty(m, dtype=torch.uint8, device=self._device)
            if m:
                self._settle()
                scratch = torch.empty(2 * m, dtype=torch.int32, device=self._device)
                call("ash_erase", self._ptr(), keys.data_ptr(), m, out.data_ptr(),
                     scratch.data_ptr(), self._stream())
                self._size_known = False
                self._tombs_ub += m
            res = out.view(torch.bool)
        return res.cpu() if host else res

    @on_device
    def active_indices(self) -> torch.Tensor:
        """All buffer indices holding an entry, ascending (hashmap.py:458-460)."""
        with self._guard.reading():
            size = self._sync_size()
            out = torch.empty(size, dtype=torch.int32, device=self._device)
            if size:
                call("ash_active_indices", self._ptr(), out.data_ptr(), self._stream())
            return out

    @on_device
    def rehash(self, new_capacity: int) -> None:
        """Rebuild at the given capacity; content preserved, indices become
        0..size-1 in ascending old-index order (hashmap.py:462-472)."""
        new_capacity = int(new_capacity)
        if new_capacity < 1:
            raise ValueError("capacity must be >= 1")
        size = self._sync_size()
        if new_capacity < size:
            raise ValueError(f"new capacity {new_capacity} is below current size {size}")
        with self._guard.writing():
            self._rehash_into(new_capacity)

    @on_device
    def clear(self) -> None:
        """Remove every entry, keep the capacity (Open3D ``clear``); the map
        is then indistinguishable from a freshly constructed one."""
        with self._guard.writing():
            call("ash_map_reset", self._ptr(), 1, self._stream())
            self._size = 0
            self._size_known = True
            self._top_ub = 0
            self._tombs_ub = 0
            self._unsettled = False  # the reset discards the pending table

    # -- content helpers (hashmap.py:476-496) ----------------------------

    @on_device
    def items_arrays(self) -> tuple:
        act = HashMap.active_indices(self).long()
        return (self._key_buf[act].clone(), *(b[act].clone() for b in self._value_bufs))

    @on_device
    def validate(self) -> None:
        """Structural invariants (hashmap.py:483-496); raises AssertionError."""
        size = self._sync_size()
        act = HashMap.active_indices(self).long()
        free = self._heap_buf[size:].long()
        assert act.numel() == size, "size counter vs active flags"
        assert int(self._active.sum().item()) == size, "size counter vs active flags"
        assert free.numel() + act.numel() == self._capacity, "heap conservation"
        both = torch.sort(torch.cat([act, free])).values
        assert torch.equal(both, torch.arange(self._capacity, device=self._device)), \
            "active/free sets must partition the index range"
        if size:
            res = HashMap.find(self, self._key_buf[act])
            assert bool(res.masks.all()), "stored key failed lookup"
            assert torch.equal(torch.sort(res.indices.long()).values, act), \
                "lookup resolved to foreign indices"
        flags = int(self._counters[_lib.CTR_FLAGS].item())
        assert flags & _lib.FLAG_TABLE_FULL == 0, "a probe wrapped the whole table"

    @on_device
    def save(self, path, metadata=None) -> None:
        """ASHL v1 snapshot, byte-compatible with the reference (hashmap.py:498-500)."""
        from .serialize import save_map
        save_map(self, path, metadata)

    @classmethod
    def load(cls, path, backend=None, threads=1, device=None):
        """Returns ``(HashMap, metadata)`` (hashmap.py:502-505)."""
        from .serialize import load_map
        return load_map(path, backend=backend, threads=threads, device=device)


class HashSet(HashMap):
    """Hash map without value buffers (hashmap.py:508-515)."""

    def __init__(self, capacity: int, key_arity: int, backend: str = "generic",
                 threads: int = 1, auto_rehash: bool = True, device=None):
        super().__init__(capacity, key_arity, value_specs=(), backend=backend,
                         threads=threads, auto_rehash=auto_rehash, device=device)
