"""CPU oracle for the spatial-hash hot path — TEST INFRASTRUCTURE ONLY.

This module is a numpy restatement of the reference package's generic
backend (``/root/reference/pkg/src/spatialhash``).  It exists to check the
CUDA product path and to time the reference algorithm on the host cores;
nothing under ``paper_2110_00511_b200/`` imports it.  Only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline leg may use it.

Parity pinning: every public function here is checked against golden
vectors produced by running the *reference itself* (``oracle/make_golden.py``
writes ``tests/golden/*.npz``; ``tests/test_oracle_golden.py`` replays them).

Algorithm map (reference file:line each function follows):

* ``lattice_hash``            hashing.py:18-43   per-dim odd multipliers, XOR, mod n
* ``row_fingerprint64``       backends.py:31-44  64-bit row fingerprint
* ``first_occurrence_mask``   backends.py:47-96  stable fingerprint sort + exact verify
* ``FreeList``                index_heap.py:14-55  heap array + top; sorted free
* ``BucketChains``            backends.py:99-178  heads/next chains; lock-step walk
* ``OracleMap``               hashmap.py:153-515 generic backend map semantics
* ``quantize``/``voxel_downsample``  geometry.py:49-76
* ``gen_keys``                bench.py:25-48
* ``candidate_blocks``        tsdf/grid.py:98-125 (+ types.py:27-31, synthetic.py:17-36)
* ``allocate_blocks_map_calls``  tsdf/grid.py:127-150
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

# ---------------------------------------------------------------------------
# hashing (hashing.py:14-43)

_LATTICE_PRIMES = (73856093, 19349669, 83492791, 49979693)
_PHI32 = 0x9E3779B1


def lattice_multipliers(arity: int) -> np.ndarray:
    """hashing.py:18-25 — first four classic primes, then odd golden-ratio
    multiples for higher dimensions."""
    if arity < 1:
        raise ValueError("key arity must be >= 1")
    out = [_LATTICE_PRIMES[d] if d < len(_LATTICE_PRIMES)
           else ((_PHI32 * (d + 1)) | 1) & 0xFFFFFFFF for d in range(arity)]
    return np.array(out, dtype=np.uint32)


def lattice_hash(keys: np.ndarray, n_buckets: int) -> np.ndarray:
    """hashing.py:28-43 — XOR of wrap-around uint32 products, mod n."""
    if n_buckets < 1:
        raise ValueError("bucket count must be >= 1")
    k = np.atleast_2d(keys)
    words = (k.view(np.uint32) if k.dtype == np.int32 else k.astype(np.uint32))
    prod = words * lattice_multipliers(k.shape[1])
    acc = np.bitwise_xor.reduce(prod, axis=1).astype(np.uint32)
    return acc % np.uint32(n_buckets)


# ---------------------------------------------------------------------------
# first-occurrence dedup (backends.py:27-96)

_FP_FINAL = np.uint64(0xD6E8FEB86659FD93)
_FP_GOLDEN = 0x9E3779B97F4A7C15
_U64 = 0xFFFFFFFFFFFFFFFF


def row_fingerprint64(keys: np.ndarray) -> np.ndarray:
    """backends.py:31-44 — per-column (k+d+1)*odd, xor-shift 31, XOR-fold,
    final multiply and xor-shift 32; all uint64 wrap-around."""
    fp = np.zeros(len(keys), dtype=np.uint64)
    for d in range(keys.shape[1]):
        odd = np.uint64(((_FP_GOLDEN * (2 * d + 1)) | 1) & _U64)
        c = keys[:, d].astype(np.uint64) + np.uint64(d + 1)
        c = c * odd
        fp ^= c ^ (c >> np.uint64(31))
    fp = fp * _FP_FINAL
    return fp ^ (fp >> np.uint64(32))


def _firsts_given_order(keys: np.ndarray, order: np.ndarray) -> np.ndarray:
    """backends.py:47-56 — with a stable row order, a group's first row is
    the lowest original position."""
    out = np.zeros(len(keys), dtype=bool)
    ordered = keys[order]
    starts = np.ones(len(keys), dtype=bool)
    starts[1:] = (ordered[1:] != ordered[:-1]).any(axis=1)
    out[order[starts]] = True
    return out


def first_occurrence_mask(keys: np.ndarray) -> np.ndarray:
    """backends.py:59-96 — True exactly at the lowest batch position of
    each distinct key row."""
    m = len(keys)
    if m == 0:
        return np.zeros(0, dtype=bool)
    if keys.shape[1] == 1:
        return _firsts_given_order(keys, np.argsort(keys[:, 0], kind="stable"))
    if m <= 4096:
        return _firsts_given_order(keys, np.lexsort(keys.T[::-1]))
    fp = row_fingerprint64(keys)
    order = np.argsort(fp, kind="stable")
    sfp = fp[order]
    run_start = np.ones(m, dtype=bool)
    run_start[1:] = sfp[1:] != sfp[:-1]
    heads = np.flatnonzero(run_start)
    out = np.zeros(m, dtype=bool)
    out[order[heads]] = True
    lengths = np.diff(np.append(heads, m))
    if lengths.max(initial=0) > 1:
        # rows in multi-row runs are equal keys or fingerprint collisions;
        # re-decide the collided ones exactly
        run_of = np.cumsum(run_start) - 1
        multi = lengths[run_of] > 1
        rows = order[multi]
        rep = order[heads][run_of[multi]]
        odd = rows[(keys[rows] != keys[rep]).any(axis=1)]
        if odd.size:
            sub = _firsts_given_order(keys[odd], np.lexsort(keys[odd].T[::-1]))
            out[odd[sub]] = True
    return out


# ---------------------------------------------------------------------------
# index heap (index_heap.py:14-55)

class HeapExhausted(RuntimeError):
    pass


class FreeList:
    """index_heap.py:14-55 — ``heap[top:]`` are free; allocate takes a
    contiguous run; free writes the *sorted* indices just below top."""

    def __init__(self, capacity: int):
        if capacity < 1:
            raise ValueError("capacity must be >= 1")
        self.capacity = capacity
        self.heap = np.arange(capacity, dtype=np.int32)
        self.top = 0

    @property
    def free_count(self) -> int:
        return self.capacity - self.top

    def allocate(self, count: int) -> np.ndarray:
        if count < 0:
            raise ValueError("count must be >= 0")
        if count > self.free_count:
            raise HeapExhausted(f"requested {count}, {self.free_count} free")
        got = self.heap[self.top:self.top + count].copy()
        self.top += count
        return got

    def free(self, idx) -> None:
        idx = np.asarray(idx, dtype=np.int32)
        if idx.size == 0:
            return
        if idx.size > self.top:
            raise ValueError("freeing more indices than were allocated")
        self.heap[self.top - idx.size:self.top] = np.sort(idx)
        self.top -= idx.size

    def free_set(self) -> np.ndarray:
        return self.heap[self.top:].copy()


# ---------------------------------------------------------------------------
# chained table (backends.py:99-220, generic backend)

class BucketChains:
    """backends.py:99-178 and 181-220 — bucket heads + per-node next links;
    nodes own a key copy and a buffer index."""

    def __init__(self, capacity: int, arity: int):
        self.n_buckets = capacity
        self.head = np.full(capacity, -1, dtype=np.int32)
        self.link = np.full(capacity, -1, dtype=np.int32)
        self.node_key = np.zeros((capacity, arity), dtype=np.int32)
        self.node_buf = np.full(capacity, -1, dtype=np.int32)
        self.node_free = np.arange(capacity, dtype=np.int32)
        self.node_top = 0

    def walk(self, keys, buckets, want_prev=False):
        """backends.py:107-133 — all chains advanced one hop per step."""
        m = len(keys)
        node = np.full(m, -1, dtype=np.int32)
        hit = np.zeros(m, dtype=bool)
        prev = np.full(m, -1, dtype=np.int32)
        cur = self.head[buckets].astype(np.int32)
        live = np.flatnonzero(cur >= 0)
        while live.size:
            at = cur[live]
            eq = (self.node_key[at] == keys[live]).all(axis=1)
            node[live[eq]] = at[eq]
            hit[live[eq]] = True
            go = live[~eq]
            prev[go] = cur[go]
            cur[go] = self.link[cur[go]]
            live = go[cur[go] >= 0]
        return (node, hit, prev) if want_prev else (node, hit)

    def add(self, keys, buckets, buf_idx) -> None:
        """backends.py:207-213 + 135-153 — take nodes off the node free
        list, then push each bucket's new nodes (batch order kept) in
        front of its existing chain."""
        k = len(buf_idx)
        if k == 0:
            return
        nodes = self.node_free[self.node_top:self.node_top + k].copy()
        self.node_top += k
        self.node_key[nodes] = keys
        self.node_buf[nodes] = buf_idx
        order = np.argsort(buckets, kind="stable")
        n_sorted, b_sorted = nodes[order], buckets[order]
        group_end = np.ones(k, dtype=bool)
        group_end[:-1] = b_sorted[1:] != b_sorted[:-1]
        nxt = np.empty(k, dtype=np.int32)
        nxt[:-1] = n_sorted[1:]
        nxt[-1] = -1
        self.link[n_sorted] = np.where(group_end, self.head[b_sorted], nxt)
        group_start = np.ones(k, dtype=bool)
        group_start[1:] = group_end[:-1]
        self.head[b_sorted[group_start]] = n_sorted[group_start]

    def drop(self, nodes, buckets, prevs) -> None:
        """backends.py:155-178 + 215-220 — unlink marked nodes (runs of
        marked nodes are skipped), then return nodes sorted to the node
        free list."""
        if nodes.size == 0:
            return
        gone = np.zeros(self.link.size, dtype=bool)
        gone[nodes] = True

        def skip_gone(start):
            out = start.copy()
            while True:
                bad = np.flatnonzero((out >= 0) & gone[np.maximum(out, 0)])
                if not bad.size:
                    return out
                out[bad] = self.link[out[bad]]

        after = skip_gone(self.link[nodes])
        keep_prev = (prevs >= 0) & ~gone[np.maximum(prevs, 0)]
        touched = np.unique(buckets)
        new_head = skip_gone(self.head[touched])
        self.link[prevs[keep_prev]] = after[keep_prev]
        self.head[touched] = new_head
        self.link[nodes] = -1
        k = nodes.size
        self.node_free[self.node_top - k:self.node_top] = np.sort(nodes)
        self.node_top -= k
        self.node_buf[nodes] = -1


# ---------------------------------------------------------------------------
# the map (hashmap.py:153-515, generic backend semantics)

class OracleCapacityError(RuntimeError):
    pass


@dataclass
class OracleResult:
    indices: np.ndarray
    masks: np.ndarray

    def __iter__(self):
        return iter((self.indices, self.masks))


def _spec(s):
    """hashmap.py:48-56 — ValueSpec coercion: (shape, dtype) or bare dtype."""
    if isinstance(s, tuple) and len(s) == 2 and isinstance(s[0], (tuple, list)):
        return tuple(int(x) for x in s[0]), np.dtype(s[1])
    if (hasattr(s, "shape") and hasattr(s, "dtype")
            and not isinstance(s, (np.dtype, type))):
        return tuple(int(x) for x in s.shape), np.dtype(s.dtype)
    return (1,), np.dtype(s)


class OracleMap:
    """Generic-backend map: key/value buffers by index, heap-dispensed
    indices, first-occurrence winners, lowest winner rank gets heap[top]."""

    def __init__(self, capacity, key_arity, value_specs=(), auto_rehash=True,
                 bucket_factor=None, backend="generic"):
        if capacity < 1:
            raise ValueError("capacity must be >= 1")
        if key_arity < 1:
            raise ValueError("key arity must be >= 1")
        if backend not in ("generic", "delegate", "integer_delegate"):
            raise ValueError(f"unknown backend {backend!r}")
        self.key_arity = int(key_arity)
        self.specs = [_spec(s) for s in value_specs]
        self.auto_rehash = auto_rehash
        # hashmap.py:187 / backends.py:230-235: delegate chains use 2c buckets
        self.delegate = backend != "generic"
        self.bucket_factor = bucket_factor or (2 if self.delegate else 1)
        self._reset(int(capacity))

    def _reset(self, capacity):
        """hashmap.py:200-210."""
        self.capacity = capacity
        self.heap = FreeList(capacity)
        self.key_buf = np.zeros((capacity, self.key_arity), dtype=np.int32)
        self.value_bufs = [np.zeros((capacity, *shape), dtype=dt)
                           for shape, dt in self.specs]
        self.active = np.zeros(capacity, dtype=bool)
        self.size = 0
        self.chains = BucketChains(capacity, self.key_arity)

    @property
    def bucket_count(self):
        return self.capacity * self.bucket_factor

    @property
    def key_buffer(self):
        return self.key_buf

    def value_buffer(self, i=0):
        return self.value_bufs[i]

    # hashmap.py:246-264
    def _keys(self, keys):
        k = np.asarray(keys)
        if k.dtype.kind == "f":
            raise ValueError("floating-point keys are not accepted; quantize to int32 first")
        if k.ndim == 1:
            if self.key_arity == 1:
                k = k.reshape(-1, 1)
            elif k.size == self.key_arity:
                k = k.reshape(1, -1)
        if k.ndim != 2 or k.shape[1] != self.key_arity:
            raise ValueError(f"keys must have shape (n, {self.key_arity}), got {k.shape}")
        if k.dtype != np.int32:
            c = k.astype(np.int32)
            if np.any(c != k):
                raise ValueError("key values do not fit in int32")
            k = c
        return np.ascontiguousarray(k)

    # hashmap.py:266-286
    def _values(self, m, values):
        if len(values) != len(self.specs):
            raise ValueError(f"expected {len(self.specs)} value batches, got {len(values)}")
        out = []
        for pos, ((shape, dt), v) in enumerate(zip(self.specs, values)):
            a = np.asarray(v)
            if a.dtype != dt:
                a = a.astype(dt)
            if a.shape[0] != m and not (m == 0 and a.size == 0):
                raise ValueError(f"value batch {pos} has length {a.shape[0]}, expected {m}")
            out.append(a.reshape((m, *shape)))
        return out

    def _lookup(self, keys, want_prev=False):
        """hashmap.py:290-298 (single worker)."""
        if self.size == 0:
            m = len(keys)
            z = np.full(m, -1, dtype=np.int32)
            f = np.zeros(m, dtype=bool)
            return (z, f, z.copy()) if want_prev else (z, f)
        b = lattice_hash(keys, self.chains.n_buckets)
        return self.chains.walk(keys, b, want_prev)

    def _grow_to(self, extra):
        """hashmap.py:311-324."""
        if self.heap.free_count >= extra:
            return
        if not self.auto_rehash:
            raise OracleCapacityError(
                f"batch needs {extra} free slots, {self.heap.free_count} available")
        cap = self.capacity
        while cap - self.size < extra:
            cap *= 2
        self._rebuild(cap)

    def _rebuild(self, capacity):
        """hashmap.py:326-332 — re-insert live rows in ascending index order."""
        live = np.flatnonzero(self.active)
        k = self.key_buf[live].copy()
        vs = [b[live].copy() for b in self.value_bufs]
        self._reset(capacity)
        if len(k):
            self._insert_like(k, vs, assoc=False)

    def _insert_delegate(self, keys):
        """hashmap.py:369-387 (delegate branch): the whole batch takes
        heap[top : top + m] (the buffer must hold size + m transiently), every
        key row is written, winner j keeps heap[top + j], the rest return to
        the heap sorted (index_heap.py:38-47) with their stale key rows."""
        m = len(keys)
        self._grow_to(m)
        all_idx = self.heap.allocate(m)
        self.key_buf[all_idx] = keys
        node, found = self._lookup(keys)
        if found.any():
            miss = np.flatnonzero(~found)
            win = miss[first_occurrence_mask(keys[miss])]
        else:
            win = np.flatnonzero(first_occurrence_mask(keys))
        widx = all_idx[win]
        self.chains.add(keys[win], lattice_hash(keys[win], self.chains.n_buckets), widx)
        loser = np.ones(m, dtype=bool)
        loser[win] = False
        self.heap.free(all_idx[loser])
        return node, found, win, widx

    def _insert_like(self, keys, vals, assoc):
        """hashmap.py:362-413 (generic branch; delegate via _insert_delegate)."""
        m = len(keys)
        idx = np.full(m, -1, dtype=np.int32)
        msk = np.zeros(m, dtype=bool)
        if m == 0:
            return OracleResult(idx, msk)
        if self.delegate:
            node, found, win, widx = self._insert_delegate(keys)
            return self._finish_insert(keys, vals, assoc, node, found, win, widx, idx, msk)
        while True:
            node, found = self._lookup(keys)
            if found.any():
                miss = np.flatnonzero(~found)
                win = miss[first_occurrence_mask(keys[miss])]
            else:
                win = np.flatnonzero(first_occurrence_mask(keys))
            if self.heap.free_count >= win.size:
                break
            self._grow_to(win.size)
        widx = self.heap.allocate(win.size)
        self.key_buf[widx] = keys[win]
        self.chains.add(keys[win], lattice_hash(keys[win], self.chains.n_buckets), widx)
        return self._finish_insert(keys, vals, assoc, node, found, win, widx, idx, msk)

    def _finish_insert(self, keys, vals, assoc, node, found, win, widx, idx, msk):
        """hashmap.py:397-413."""
        if vals is not None:
            for buf, v in zip(self.value_bufs, vals):
                if widx.size:
                    buf[widx] = v[win]
        self.active[widx] = True
        self.size += win.size
        idx[win] = widx
        msk[win] = True
        if assoc:
            fp = np.flatnonzero(found)
            idx[fp] = self.chains.node_buf[node[fp]]
            msk[fp] = True
        return OracleResult(idx, msk)

    def insert(self, keys, *values):
        keys = self._keys(keys)
        return self._insert_like(keys, self._values(len(keys), values), assoc=False)

    def activate(self, keys):
        return self._insert_like(self._keys(keys), None, assoc=True)

    def find(self, keys):
        """hashmap.py:415-429."""
        keys = self._keys(keys)
        m = len(keys)
        idx = np.full(m, -1, dtype=np.int32)
        msk = np.zeros(m, dtype=bool)
        if m == 0:
            return OracleResult(idx, msk)
        node, found = self._lookup(keys)
        hit = np.flatnonzero(found)
        idx[hit] = self.chains.node_buf[node[hit]]
        msk[hit] = True
        return OracleResult(idx, msk)

    def erase(self, keys):
        """hashmap.py:431-456."""
        keys = self._keys(keys)
        m = len(keys)
        out = np.zeros(m, dtype=bool)
        if m == 0:
            return out
        node, found, prev = self._lookup(keys, want_prev=True)
        fpos = np.flatnonzero(found)
        if not fpos.size:
            return out
        hit = fpos[first_occurrence_mask(keys[fpos])]
        bidx = self.chains.node_buf[node[hit]].copy()
        self.chains.drop(node[hit], lattice_hash(keys[hit], self.chains.n_buckets), prev[hit])
        self.heap.free(bidx)
        self.active[bidx] = False
        self.size -= hit.size
        out[hit] = True
        return out

    def active_indices(self):
        return np.flatnonzero(self.active).astype(np.int32)

    def rehash(self, new_capacity):
        """hashmap.py:462-472."""
        new_capacity = int(new_capacity)
        if new_capacity < 1:
            raise ValueError("capacity must be >= 1")
        if new_capacity < self.size:
            raise ValueError(f"new capacity {new_capacity} is below current size {self.size}")
        self._rebuild(new_capacity)

    def items_arrays(self):
        live = np.flatnonzero(self.active)
        return (self.key_buf[live].copy(), *(b[live].copy() for b in self.value_bufs))


class OracleSet(OracleMap):
    def __init__(self, capacity, key_arity, auto_rehash=True, backend="generic"):
        super().__init__(capacity, key_arity, (), auto_rehash, backend=backend)


# ---------------------------------------------------------------------------
# geometry (geometry.py:49-76)

def quantize(positions, cell: float) -> np.ndarray:
    """geometry.py:49-56 — float64 true division, floor, int32 range check."""
    if cell <= 0:
        raise ValueError("cell size must be > 0")
    q = np.floor(np.asarray(positions, dtype=np.float64) / cell)
    if q.size and (q.min() < -(2 ** 31) or q.max() >= 2 ** 31):
        raise ValueError("quantized coordinates exceed int32 range")
    return q.astype(np.int32)


def voxel_downsample(points, voxel_size: float):
    """geometry.py:59-76 — HashSet insert of the quantized coordinates;
    representatives are the first occurrences, ascending."""
    pos = np.asarray(points, dtype=np.float64).reshape(-1, 3)
    coords = quantize(pos, voxel_size)
    if len(coords) == 0:
        return coords, np.zeros(0, dtype=np.int64)
    s = OracleSet(len(coords), 3)
    sel = np.flatnonzero(s.insert(coords).masks)
    return coords[sel], sel


# ---------------------------------------------------------------------------
# synthetic workloads

def gen_keys(count: int, uniqueness: float, kind: str = "int3", seed: int = 0):
    """bench.py:25-48 — ceil(rho*count) distinct keys drawn from
    [-2^20, 2^20)^arity (int3) plus uniform duplicates, shuffled."""
    if not 0 < uniqueness <= 1:
        raise ValueError("uniqueness must be in (0, 1]")
    arity = {"int3": 3, "int1": 1}[kind]
    n_unique = int(np.ceil(uniqueness * count))
    rng = np.random.default_rng(seed)
    lo, hi = ((-(2 ** 20), 2 ** 20) if arity == 3 else (-(2 ** 31), 2 ** 31))
    pool = np.zeros((0, arity), dtype=np.int64)
    while len(pool) < n_unique:
        draw = rng.integers(lo, hi, size=(max(n_unique, 64), arity))
        pool = np.unique(np.concatenate([pool, draw]), axis=0)
    pool = pool[rng.permutation(len(pool))[:n_unique]]
    extra = pool[rng.integers(0, n_unique, size=count - n_unique)]
    batch = np.concatenate([pool, extra])
    rng.shuffle(batch, axis=0)
    return batch.astype(np.int32)


@dataclass(frozen=True)
class Camera:
    """tsdf/types.py:9-31 — pinhole intrinsics."""
    fx: float
    fy: float
    cx: float
    cy: float
    width: int
    height: int

    def unproject(self, u, v, z):
        x = (np.asarray(u) - self.cx) / self.fx * z
        y = (np.asarray(v) - self.cy) / self.fy * z
        return np.stack([x, y, np.broadcast_to(z, np.shape(x))], axis=-1)


def scaled_camera(width: int, height: int) -> Camera:
    """cli.py:125-130 scaling of synthetic.DEFAULT_INTRINSICS (250, 250,
    159.5, 119.5, 320x240) to another width."""
    s = width / 320
    return Camera(250.0 * s, 250.0 * s, (width - 1) / 2, (height - 1) / 2, width, height)


def plane_depth(cam: Camera, z: float = 1.0) -> np.ndarray:
    """tsdf/synthetic.py:17-19."""
    return np.full((cam.height, cam.width), float(z))


def sphere_depth(cam: Camera, center=(0.0, 0.0, 1.0), radius=0.3) -> np.ndarray:
    """tsdf/synthetic.py:22-36 — ray/sphere first hit, 0 where missed."""
    uu, vv = np.meshgrid(np.arange(cam.width), np.arange(cam.height))
    d = cam.unproject(uu.ravel(), vv.ravel(), 1.0)
    d /= np.linalg.norm(d, axis=1, keepdims=True)
    c = np.asarray(center, dtype=np.float64)
    b = d @ c
    disc = b * b - (c @ c - radius * radius)
    hit = disc >= 0
    t = np.where(hit, b - np.sqrt(np.maximum(disc, 0.0)), 0.0)
    hit &= t > 0
    return np.where(hit, t * d[:, 2], 0.0).reshape(cam.height, cam.width)


def candidate_blocks(depth, cam: Camera, pose, block_size: float, trunc: float,
                     depth_min=0.2, depth_max=3.0) -> np.ndarray:
    """tsdf/grid.py:98-125 (ray mode) + grid.py:24-27 block_of: samples at
    half-block spacing within +-trunc of the surface, floor(x / block)."""
    depth = np.asarray(depth, dtype=np.float64)
    ok = (depth > 0) & (depth >= depth_min) & (depth <= depth_max)
    v, u = np.nonzero(ok)
    if v.size == 0:
        return np.zeros((0, 3), dtype=np.int32)
    z = depth[v, u]
    rays = cam.unproject(u, v, 1.0)
    pose = np.asarray(pose, dtype=np.float64)
    rot, trans = pose[:3, :3], pose[:3, 3]
    step = block_size / 2
    n = int(np.ceil(2 * trunc / step)) + 1
    t = np.minimum(np.arange(n) * step, 2 * trunc)
    dep = np.maximum(z[:, None] - trunc + t[None, :], 1e-6)
    pts = rays[:, None, :] * dep[..., None]
    world = pts.reshape(-1, 3) @ rot.T + trans
    return np.floor(world / block_size).astype(np.int32)


def allocate_blocks_map_calls(global_map: OracleMap, coords: np.ndarray):
    """tsdf/grid.py:136-150 — local dedup map, global activate + find,
    local values hold the global index.  Returns (gi, local_map, li, lmask)."""
    local = OracleMap(len(coords), 3, [np.int32])
    li, lmask = local.activate(coords)
    surv = coords[lmask]
    global_map.activate(surv)
    gi, gmask = global_map.find(surv)
    assert bool(gmask.all())
    local.value_buffer(0)[li[lmask], 0] = gi
    return gi, local, li, lmask
