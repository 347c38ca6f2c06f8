"""The reference property suite (pkg/tests/test_hashmap_properties.py) with
the CUDA map under test and the oracle as the sequential reference; indices
are compared exactly, not just masks and content."""
import numpy as np
import pytest
from hypothesis import HealthCheck, given, settings, strategies as st

from conftest import to_np

pytestmark = pytest.mark.gpu

key_batches = st.lists(st.tuples(st.integers(-6, 6), st.integers(-6, 6), st.integers(-6, 6)),
                       min_size=0, max_size=40)
op_sequences = st.lists(st.tuples(st.sampled_from(["insert", "erase", "find", "activate", "rehash"]),
                                  key_batches), min_size=1, max_size=30)
SETTINGS = dict(deadline=None, suppress_health_check=[HealthCheck.function_scoped_fixture])


@pytest.fixture(scope="module")
def mods(cuda_ok):
    import paper_2110_00511_b200 as ash
    from oracle import ash_oracle as O
    return ash, O


def _value_for(key):
    return np.float32(key[0] * 100 + key[1] * 10 + key[2])


@settings(max_examples=120, **SETTINGS)
@given(op_sequences)
def test_op_sequences_match_oracle_exactly(mods, ops):
    ash, O = mods
    m = ash.HashMap(4, 3, value_specs=[np.float32], device="cuda")
    ref = O.OracleMap(4, 3, [np.float32])
    for op, batch in ops:
        keys = np.asarray(batch, np.int32).reshape(-1, 3)
        vals = np.array([_value_for(k) for k in batch], np.float32).reshape(-1, 1)
        if op == "insert":
            a, b = m.insert(keys, vals), ref.insert(keys, vals)
        elif op == "activate":
            a, b = m.activate(keys), ref.activate(keys)
        elif op == "find":
            a, b = m.find(keys), ref.find(keys)
        elif op == "erase":
            assert np.array_equal(to_np(m.erase(keys)), ref.erase(keys))
            continue
        else:
            c = max(2 * ref.size, ref.size + len(batch), 4)
            m.rehash(c)
            ref.rehash(c)
            continue
        assert np.array_equal(to_np(a.indices), b.indices)
        assert np.array_equal(to_np(a.masks), b.masks)
        assert m.size == ref.size and m.capacity == ref.capacity
    assert to_np(m.key_buffer).tobytes() == ref.key_buffer.tobytes()
    assert to_np(m.value_buffer(0)).tobytes() == ref.value_buffer(0).tobytes()
    m.validate()


@settings(max_examples=60, **SETTINGS)
@given(key_batches)
def test_heap_conservation_and_rehash_content(mods, batch):
    ash, O = mods
    keys = np.asarray(batch, np.int32).reshape(-1, 3)
    m = ash.HashMap(max(len(batch), 1), 3, value_specs=[np.float32], device="cuda")
    m.insert(keys, np.arange(len(batch), dtype=np.float32).reshape(-1, 1))
    assert m._heap.free_count + m.size == m.capacity
    before = [to_np(x) for x in m.items_arrays()]
    m.rehash(2 * m.capacity + 1)
    after = [to_np(x) for x in m.items_arrays()]
    assert all(np.array_equal(x, y) for x, y in zip(before, after))
    m.erase(keys[: len(batch) // 2])
    assert m._heap.free_count + m.size == m.capacity
    m.validate()


def test_dedup_count_formula(mods, rng):
    # test_hashmap_properties.py:113-126
    ash, _ = mods
    m = ash.HashMap(512, 3, value_specs=[np.float32], device="cuda")
    seen = set()
    for _ in range(30):
        n = int(rng.integers(1, 120))
        keys = rng.integers(-4, 4, size=(n, 3)).astype(np.int32)
        unique = {tuple(k) for k in keys}
        res = m.insert(keys, np.ones((n, 1), np.float32))
        assert int(res.masks.sum()) == len(unique - seen)
        seen |= unique
        assert m.size == len(seen)


def test_dedup_1000_cases(mods):
    # tests/test_acceptance.py:29-46 (correctness part; the 60 s budget is CPU)
    ash, _ = mods
    rng = np.random.default_rng(101)
    for case in range(1000):
        c = int(10 ** rng.uniform(0, 5))
        rho = float(rng.uniform(0.01, 1.0))
        n_unique = max(1, int(rho * c))
        pool = rng.integers(-2 ** 20, 2 ** 20, size=(n_unique, 3)).astype(np.int32)
        keys = pool[rng.integers(0, n_unique, size=c)]
        oracle = len(np.unique(keys, axis=0))
        s = ash.HashSet(c, 3, backend=("generic", "delegate")[case % 2], device="cuda")
        res = s.insert(keys)
        assert int(res.masks.sum()) == oracle == s.size, (case, c, rho)
