"""Synthetic inputs for the benchmark configurations (BASELINE.json configs).

``int3_batch`` reproduces the *distribution* of the reference generator
(bench.py:25-48: ceil(rho*n) distinct keys uniform in [-2^20, 2^20)^3, the
rest uniform duplicates of the pool, shuffled) without its O(n log n)
``np.unique`` loop: distinct keys come from a bijection on 63-bit counters
(three 21-bit fields), so 10M keys take well under a second.  It is also the
counter-based generator SURVEY §8(d) specifies for the partitioned stream.
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


def c5_step_batches(start: int, size: int, total: int, seed: int = 0, device=None):
    """configs[4] stream: a step inserts pool keys
    [start, start + size) and finds ``size`` keys, half drawn from the keys
    inserted so far and half from never-inserted pool indices >= total."""
    import torch
    g = torch.Generator(device=device).manual_seed(seed * 1000003 + start)
    ins = torch.arange(start, start + size, device=device)
    half = size // 2
    hit = torch.randint(0, start + size, (half,), generator=g, device=device)
    miss = torch.randint(total, 2 * total, (size - half,), generator=g, device=device)
    q = torch.cat([hit, miss])
    q = q[torch.randperm(size, generator=g, device=device)]
    return keys_from_counters_torch(ins, seed), keys_from_counters_torch(q, seed)
