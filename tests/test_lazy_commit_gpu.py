"""Deferred slot-state commit (ash_insert_lazy / ash_settle).

A large insert leaves its winners PENDING|pos in the table; finds and
lattice finds resolve them from the rank words, every mutating call settles
first.  Every op sequence must give bit-identical results to the eager
commit (the sweep inside the insert) and to the oracle."""
import contextlib

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ash(cuda_ok):
    import paper_2110_00511_b200 as ash
    return ash


@pytest.fixture(scope="module", autouse=True)
def sweep_small_tables(cuda_ok):
    """These maps are small enough to stay in the L2, where inserts skip the
    table sweep; the tests exercise the sweep, so allow it for every size."""
    from paper_2110_00511_b200 import _lib
    _lib.lib.ash_set_sweep_table_min(0)
    yield
    _lib.lib.ash_set_sweep_table_min(-1)


@pytest.fixture(autouse=True)
def lazy_default():
    """The deferred commit is opt-in (ASH_LAZY_COMMIT=1); these tests turn it on."""
    from paper_2110_00511_b200 import hashmap as hm
    old = hm.LAZY_COMMIT
    hm.LAZY_COMMIT = True
    yield
    hm.LAZY_COMMIT = old


@contextlib.contextmanager
def eager():
    from paper_2110_00511_b200 import hashmap as hm
    old = hm.LAZY_COMMIT
    hm.LAZY_COMMIT = False
    try:
        yield
    finally:
        hm.LAZY_COMMIT = old


def pair(ash, *args, **kw):
    return ash.HashMap(*args, device="cuda", **kw), ash.HashMap(*args, device="cuda", **kw)


def same(a, b):
    if not isinstance(a, torch.Tensor):  # BatchResult (a tensor's .indices is a method)
        return torch.equal(a.indices, b.indices) and torch.equal(a.masks, b.masks)
    return torch.equal(a, b)


def test_pending_slots_resolve_in_find(ash):
    from oracle.ash_oracle import OracleMap
    rng = np.random.default_rng(3)
    keys = torch.from_numpy(rng.integers(-3000, 3000, size=(200_000, 3)).astype(np.int32)).cuda()
    vals = torch.rand((200_000, 2), device="cuda")
    lazy, ref = pair(ash, 200_000, 3, [((2,), np.float32)])
    r1 = lazy.insert(keys, vals)
    assert lazy._unsettled  # the sweep was deferred
    # the table really holds PENDING states until settled
    st = lazy._slots.view(-1, 4)[:, 3].to(torch.int64) & 0xFFFFFFFF
    pend = (st >> 30) == 2
    assert int(pend.sum()) > 0
    with eager():
        r2 = ref.insert(keys, vals)
    assert same(r1, r2)
    q = torch.from_numpy(rng.integers(-3500, 3500, size=(300_000, 3)).astype(np.int32)).cuda()
    assert same(lazy.find(q), ref.find(q))
    assert lazy._unsettled  # finds do not settle
    om = OracleMap(200_000, 3, [((2,), np.float32)])
    om.insert(keys.cpu().numpy(), vals.cpu().numpy())
    assert np.array_equal(lazy.find(q).indices.cpu().numpy(), om.find(q.cpu().numpy()).indices)
    nb1 = ash.radius_neighbors(lazy, q[:5000], 1)
    nb2 = ash.radius_neighbors(ref, q[:5000], 1)
    assert same(nb1, nb2)
    lazy.validate()


@pytest.mark.parametrize("op", ["insert", "activate", "erase", "rehash", "reserve"])
def test_mutation_after_deferred_commit(ash, op):
    rng = np.random.default_rng(7)
    k1 = torch.from_numpy(rng.integers(-2000, 2000, size=(150_000, 3)).astype(np.int32)).cuda()
    k2 = torch.from_numpy(rng.integers(-2200, 2200, size=(150_000, 3)).astype(np.int32)).cuda()
    v1 = torch.rand((150_000, 1), device="cuda")
    v2 = torch.rand((150_000, 1), device="cuda")
    lazy, ref = pair(ash, 150_000, 3, [np.float32])
    lazy.insert(k1, v1)
    with eager():
        ref.insert(k1, v1)
        if op == "insert":
            a, b = lazy.insert(k2, v2), ref.insert(k2, v2)
        elif op == "activate":
            a, b = lazy.activate(k2), ref.activate(k2)
        elif op == "erase":
            a, b = lazy.erase(k2), ref.erase(k2)
        elif op == "rehash":
            lazy.rehash(400_000)
            ref.rehash(400_000)
            a, b = lazy.find(k2), ref.find(k2)
        else:
            lazy.reserve(600_000)
            ref.reserve(600_000)
            a, b = lazy.insert(k2, v2), ref.insert(k2, v2)
    assert same(a, b)
    assert lazy.size == ref.size
    assert same(lazy.find(k1), ref.find(k1)) and same(lazy.find(k2), ref.find(k2))
    assert torch.equal(lazy.active_indices(), ref.active_indices())
    lazy.validate()


def test_deferred_commit_over_a_dirty_heap(ash):
    """Frees put sorted indices back above top: the resolution must read
    heap[top + rank] instead of top + rank."""
    rng = np.random.default_rng(11)
    base = torch.from_numpy(rng.integers(-5000, 5000, size=(120_000, 3)).astype(np.int32)).cuda()
    lazy, ref = pair(ash, 120_000, 3, [np.float32])
    v = torch.rand((120_000, 1), device="cuda")
    with eager():
        ref.insert(base, v)
        ref.erase(base[::3])
    lazy.insert(base, v)
    lazy.erase(base[::3])
    new = torch.from_numpy(rng.integers(-9000, 9000, size=(120_000, 3)).astype(np.int32)).cuda()
    a = lazy.insert(new, v)
    assert lazy._unsettled
    with eager():
        b = ref.insert(new, v)
    assert same(a, b)
    allk = torch.cat([base, new])
    assert same(lazy.find(allk), ref.find(allk))
    assert torch.equal(lazy.value_buffer(0), ref.value_buffer(0))
    lazy.validate()


@pytest.mark.parametrize("arity", [1, 2, 5])
def test_deferred_commit_other_arities(ash, arity):
    rng = np.random.default_rng(arity)
    keys = torch.from_numpy(rng.integers(-40, 40, size=(100_000, arity)).astype(np.int32)).cuda()
    lazy, ref = pair(ash, 100_000, arity)
    a = lazy.insert(keys)
    with eager():
        b = ref.insert(keys)
    assert same(a, b)
    q = torch.from_numpy(rng.integers(-45, 45, size=(100_000, arity)).astype(np.int32)).cuda()
    assert same(lazy.find(q), ref.find(q))
    lazy.validate()


def test_clear_discards_pending(ash):
    rng = np.random.default_rng(5)
    keys = torch.from_numpy(rng.integers(-9000, 9000, size=(100_000, 3)).astype(np.int32)).cuda()
    m = ash.HashMap(100_000, 3, device="cuda")
    r1 = m.insert(keys)
    m.clear()
    assert not m._unsettled
    r2 = m.insert(keys)
    assert same(r1, r2)
    f = m.find(keys)
    assert bool(f.masks.all()) and torch.equal(f.indices[r2.masks], r2.indices[r2.masks])
