"""Larger randomized op streams against the oracle, chosen to cross every
commit strategy: the TMA-staged commit with 4-, 16- and 32-byte value rows,
the plain commit (arity > 3, two value buffers), the table-sweep slot commit
(batches with >= n_buckets / 5 winners) with an identity and a freed
(non-identity) heap, tombstone rebuilds, growth, and the delegate backend.
Indices are compared exactly."""
import numpy as np
import pytest

import golden_replay as G

pytestmark = pytest.mark.gpu

CASES = [
    # (arity, value specs, backend, key span, steps)
    (3, [np.float32], "generic", 4000, 24),
    (3, [((4,), np.float32)], "generic", 30000, 20),
    (3, [((8,), np.float32)], "generic", 30000, 16),
    (4, [np.float32], "generic", 60, 16),
    (3, [np.float32, ((3,), np.int16)], "generic", 30000, 16),
    (2, [np.int64], "delegate", 400, 16),
]


@pytest.fixture(scope="module")
def mods(cuda_ok):
    import paper_2110_00511_b200 as ash
    from oracle import ash_oracle as O
    return ash, O


def _values(rng, specs, n):
    out = []
    for s in specs:
        shape, dt = (s if isinstance(s, tuple) else ((1,), s))
        if np.dtype(dt).kind == "f":
            out.append(rng.random((n, *shape)).astype(dt))
        else:
            out.append(rng.integers(-30000, 30000, size=(n, *shape)).astype(dt))
    return out


@pytest.mark.parametrize("case", range(len(CASES)))
def test_stream_vs_oracle(mods, case):
    ash, O = mods
    arity, specs, backend, span, steps = CASES[case]
    rng = np.random.default_rng(900 + case)
    cap = 150_000
    g = ash.HashMap(cap, arity, specs, backend=backend, device="cuda")
    o = O.OracleMap(cap, arity, specs, backend=backend)
    for step in range(steps):
        op = rng.choice(["insert", "insert", "activate", "erase", "find"])
        n = int(rng.integers(0, 250_000))
        keys = rng.integers(-span, span, size=(n, arity)).astype(np.int32)
        if op == "insert":
            vals = _values(rng, specs, n)
            a, b = g.insert(keys, *vals), o.insert(keys, *vals)
        elif op == "activate":
            a, b = g.activate(keys), o.activate(keys)
        elif op == "find":
            a, b = g.find(keys), o.find(keys)
        else:
            G.eq(g.erase(keys[: n // 2]), o.erase(keys[: n // 2]), f"step {step} erase")
            continue
        G.eq(a.indices, b.indices, f"case {case} step {step} {op} idx")
        G.eq(a.masks, b.masks, f"case {case} step {step} {op} mask")
        assert g.size == o.size and g.capacity == o.capacity, (step, g.size, o.size)
    G.eq(g.active_indices(), o.active_indices(), "active")
    G.bytes_eq(g.key_buffer, o.key_buffer, "key rows")
    for i in range(len(specs)):
        G.bytes_eq(g.value_buffer(i), o.value_buffer(i), f"value buffer {i}")
    g.validate()
