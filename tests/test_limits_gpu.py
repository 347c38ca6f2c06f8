"""Edge cases at the limits: key words equal to the slot-state sentinels
(EMPTY 0xFFFFFFFF = -1, TOMBSTONE 0xFFFFFFFE = -2, the PENDING bit
0x80000000 = INT32_MIN), batch lengths at the scan-tile and warp boundaries,
capacity 1 with growth, and the single-map table limit.  Exact against the
oracle."""
import itertools

import numpy as np
import pytest

import golden_replay as G

pytestmark = pytest.mark.gpu

WORDS = [-2 ** 31, -2 ** 31 + 1, -2, -1, 0, 1, 2 ** 31 - 1]


@pytest.fixture(scope="module")
def mods(cuda_ok):
    import paper_2110_00511_b200 as ash
    from oracle import ash_oracle as O
    return ash, O


@pytest.mark.parametrize("arity", [1, 2, 3, 4])
def test_sentinel_valued_key_words(mods, arity):
    ash, O = mods
    combos = np.array(list(itertools.product(WORDS, repeat=arity)), dtype=np.int32)
    rng = np.random.default_rng(arity)
    batch = np.concatenate([combos, combos[rng.integers(0, len(combos), size=len(combos))]])
    batch = batch[rng.permutation(len(batch))]
    vals = rng.random((len(batch), 1)).astype(np.float32)
    g = ash.HashMap(len(combos) + 8, arity, [np.float32], device="cuda")
    o = O.OracleMap(len(combos) + 8, arity, [np.float32])
    a, b = g.insert(batch, vals), o.insert(batch, vals)
    G.eq(a.indices, b.indices, "insert idx")
    G.eq(a.masks, b.masks, "insert masks")
    assert g.size == len(combos)
    G.eq(g.find(combos[::-1].copy()).indices, o.find(combos[::-1].copy()).indices, "find")
    half = combos[::2].copy()
    G.eq(g.erase(half), o.erase(half), "erase")
    G.eq(g.activate(batch).indices, o.activate(batch).indices, "activate after erase")
    G.eq(g.active_indices(), o.active_indices(), "active")
    G.bytes_eq(g.key_buffer, o.key_buffer, "key rows")
    G.bytes_eq(g.value_buffer(0), o.value_buffer(0), "values")
    g.validate()


@pytest.mark.parametrize("n", [1, 31, 32, 33, 255, 256, 2047, 2048, 2049, 4095, 4097])
def test_batch_lengths_at_warp_and_tile_boundaries(mods, n):
    ash, O = mods
    rng = np.random.default_rng(n)
    keys = rng.integers(-40, 40, size=(n, 3)).astype(np.int32)
    g = ash.HashMap(64, 3, device="cuda")
    o = O.OracleMap(64, 3)
    for op in ("insert", "activate", "find", "erase", "insert"):
        k = keys if op != "erase" else keys[: max(1, n // 3)].copy()
        a, b = getattr(g, op)(k), getattr(o, op)(k)
        if op == "erase":
            G.eq(a, b, f"{n} erase")
        else:
            G.eq(a.indices, b.indices, f"{n} {op}")
        assert g.capacity == o.capacity and g.size == o.size


def test_capacity_one_grows_by_doubling(mods):
    ash, O = mods
    g, o = ash.HashMap(1, 2, device="cuda"), O.OracleMap(1, 2)
    for step in range(6):
        k = np.array([[step, i] for i in range(3 * step + 1)], dtype=np.int32)
        G.eq(g.insert(k).indices, o.insert(k).indices, f"step {step}")
        assert g.capacity == o.capacity
    G.eq(g.active_indices(), o.active_indices(), "active")


def test_table_limit_is_a_value_error(mods):
    ash, _ = mods
    with pytest.raises(ValueError, match="2\\^30"):
        ash.HashMap(800_000_000, 3, device="cuda")  # 1.2e9 slots > 2^30
