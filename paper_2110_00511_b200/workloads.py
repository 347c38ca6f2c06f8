"""Synthetic inputs for the benchmark configurations (BASELINE.json configs).

Host-only numpy (torch is imported inside the device helpers); importing this
module does not load libash.so, so the CPU reference arm can use it.

* ``gen_keys``: the reference generator (bench.py:25-48), output for output,
  with a faster but order-identical dedup of the distinct pool.
* ``int3_batch``: the same *distribution* from a bijection on 63-bit
  counters (three 21-bit fields); the partitioned bench's per-rank slices.
* ``keys_from_counters[_torch]`` / ``c5_step_*``: the counter-based
  generator SURVEY §8(d) specifies for the configs[4] stream.
* ``sphere_points``: the configs[2] cloud.
"""
from __future__ import annotations

import numpy as np

_MASK63 = (1 << 63) - 1
_M1 = 0x5DEECE66D2F0A6B5 & _MASK63 | 1
_M2 = 0x2545F4914F6CDD1D & _MASK63 | 1


def mix63(x: np.ndarray, seed: int = 0) -> np.ndarray:
    """Bijection on [0, 2^63): odd multiplies and xorshifts mod 2^63."""
    m = np.uint64(_MASK63)
    x = (x.astype(np.uint64) + np.uint64((seed * 0x9E3779B97F4A7C15) & _MASK63)) & m
    x = (x * np.uint64(_M1)) & m
    x ^= x >> np.uint64(29)
    x = (x * np.uint64(_M2)) & m
    x ^= x >> np.uint64(32)
    x = (x * np.uint64(_M1)) & m
    x ^= x >> np.uint64(27)
    return x


def keys_from_counters(counters: np.ndarray, seed: int = 0) -> np.ndarray:
    """Distinct counters -> distinct int3 keys in [-2^20, 2^20)^3."""
    u = mix63(np.asarray(counters, dtype=np.uint64), seed)
    f = np.uint64(0x1FFFFF)
    out = np.empty((len(u), 3), dtype=np.int32)
    out[:, 0] = (u & f).astype(np.int64) - (1 << 20)
    out[:, 1] = ((u >> np.uint64(21)) & f).astype(np.int64) - (1 << 20)
    out[:, 2] = ((u >> np.uint64(42)) & f).astype(np.int64) - (1 << 20)
    return out


KEY_RANGE_3D = 1 << 20  # reference bench.py:22


def gen_keys(count: int, uniqueness: float, kind: str = "int3", seed: int = 0) -> np.ndarray:
    """The reference generator, output for output (bench.py:25-48).

    Same draws from ``default_rng(seed)`` in the same order; the only change
    is the dedup of the distinct pool: the reference's ``np.unique(axis=0)``
    sorts int64 rows lexicographically, which for int3 rows in
    [-2^20, 2^20)^3 is the order of the packed 63-bit code
    ``(x+2^20)<<42 | (y+2^20)<<21 | (z+2^20)``, so a 1-D sorted unique of
    the codes gives the identical pool (10M keys: ~1-2 s instead of 15-32 s).
    Pinned against the reference at C1/C2 sizes by
    ``tests/golden/fullsize_sha.json`` (``oracle/make_fullsize_golden.py``).
    """
    if not 0 < uniqueness <= 1:
        raise ValueError("uniqueness must be in (0, 1]")
    if kind not in ("int3", "int1"):
        raise ValueError("key kind must be one of ['int1', 'int3']")
    arity = 3 if kind == "int3" else 1
    n_unique = int(np.ceil(uniqueness * count))
    rng = np.random.default_rng(seed)
    if arity == 3:
        off = np.int64(KEY_RANGE_3D)
        pool = np.zeros(0, dtype=np.int64)
        while len(pool) < n_unique:
            d = rng.integers(-KEY_RANGE_3D, KEY_RANGE_3D, size=(max(n_unique, 64), 3)) + off
            code = (d[:, 0] << np.int64(42)) | (d[:, 1] << np.int64(21)) | d[:, 2]
            pool = _sorted_unique(np.concatenate([pool, code]))
    else:
        pool = np.zeros(0, dtype=np.int64)
        while len(pool) < n_unique:
            d = rng.integers(-(2 ** 31), 2 ** 31, size=(max(n_unique, 64), 1))
            pool = _sorted_unique(np.concatenate([pool, d[:, 0]]))
    pool = pool[rng.permutation(len(pool))[:n_unique]]
    dup = pool[rng.integers(0, n_unique, size=count - n_unique)]
    batch = np.concatenate([pool, dup])
    # a 1-D shuffle of the codes draws the same swaps as the reference's
    # row shuffle (Generator.shuffle along axis 0), so the order is identical
    rng.shuffle(batch)
    if arity == 1:
        return batch.astype(np.int32)[:, None]
    f = np.int64(0x1FFFFF)
    out = np.empty((count, 3), dtype=np.int32)
    out[:, 0] = (batch >> np.int64(42)) - off
    out[:, 1] = ((batch >> np.int64(21)) & f) - off
    out[:, 2] = (batch & f) - off
    return out


def _sorted_unique(a: np.ndarray) -> np.ndarray:
    a = np.sort(a)
    keep = np.ones(len(a), dtype=bool)
    keep[1:] = a[1:] != a[:-1]
    return a[keep]


def int3_batch(count: int, uniqueness: float, seed: int = 0) -> np.ndarray:
    """``count`` int3 keys with exactly ceil(uniqueness*count) distinct ones."""
    if not 0 < uniqueness <= 1:
        raise ValueError("uniqueness must be in (0, 1]")
    n_unique = int(np.ceil(uniqueness * count))
    rng = np.random.default_rng(seed)
    pool = keys_from_counters(np.arange(n_unique, dtype=np.uint64), seed)
    dup = pool[rng.integers(0, n_unique, size=count - n_unique)]
    batch = np.concatenate([pool, dup])
    return batch[rng.permutation(count)]


def sphere_points(count: int, seed: int = 0) -> np.ndarray:
    """C3: unit-sphere surface cloud, float64."""
    d = np.random.default_rng(seed).normal(size=(count, 3))
    d /= np.linalg.norm(d, axis=1, keepdims=True)
    return d


def _signed64(c: int) -> int:
    return c - (1 << 64) if c >= 1 << 63 else c


def keys_from_counters_torch(counters, seed: int = 0):
    """Device twin of ``keys_from_counters`` (torch int64 arithmetic wraps
    mod 2^64; masking to 63 bits keeps every shift logical), so the 400M-key
    C5 stream is generated in HBM instead of crossing PCIe."""
    import torch
    m = (1 << 63) - 1
    x = (counters.to(torch.int64) + ((seed * 0x9E3779B97F4A7C15) & m)) & m
    x = (x * _signed64(_M1)) & m
    x ^= x >> 29
    x = (x * _signed64(_M2)) & m
    x ^= x >> 32
    x = (x * _signed64(_M1)) & m
    x ^= x >> 27
    f = 0x1FFFFF
    return torch.stack([(x & f) - (1 << 20), ((x >> 21) & f) - (1 << 20),
                        ((x >> 42) & f) - (1 << 20)], dim=1).to(torch.int32)


def c5_step_counters(start: int, size: int, total: int, seed: int = 0, device=None):
    """configs[4] stream as pool counters: a step inserts pool
    keys [start, start + size) and finds ``size`` keys, half drawn from the
    keys inserted so far and half from never-inserted pool indices >= total.
    With all-new keys on a fresh heap, the key of counter c gets buffer
    index c, so the counters are also the expected indices."""
    import torch
    g = torch.Generator(device=device).manual_seed(seed * 1000003 + start)
    ins = torch.arange(start, start + size, device=device)
    half = size // 2
    hit = torch.randint(0, start + size, (half,), generator=g, device=device)
    miss = torch.randint(total, 2 * total, (size - half,), generator=g, device=device)
    q = torch.cat([hit, miss])
    q = q[torch.randperm(size, generator=g, device=device)]
    return ins, q


def c5_step_batches(start: int, size: int, total: int, seed: int = 0, device=None):
    """The keys of ``c5_step_counters``."""
    ins, q = c5_step_counters(start, size, total, seed, device)
    return keys_from_counters_torch(ins, seed), keys_from_counters_torch(q, seed)
