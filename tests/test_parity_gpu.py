"""CUDA map vs golden vectors recorded from the reference, and vs the CPU
oracle on seeded random inputs.  Bit-exact: indices, masks, buffer bytes."""
import numpy as np
import pytest

import golden_replay as G
from conftest import to_np

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ash(cuda_ok):
    import paper_2110_00511_b200 as ash
    return ash


@pytest.fixture(scope="module")
def O():
    from oracle import ash_oracle
    return ash_oracle


def _mk(ash):
    return lambda cap, ar, specs: ash.HashMap(cap, ar, specs, device="cuda")


def test_trace_appendix_a(ash):
    G.replay_trace(_mk(ash))


def test_c1_insert_find(ash):
    G.replay_c1(_mk(ash))


def test_bindings_parity_cases(ash):
    G.replay_bindings(_mk(ash))


def test_random_op_sequences(ash):
    G.replay_random_ops(_mk(ash))


def test_random_op_sequences_delegate(ash):
    G.replay_random_ops(lambda c, a, sp: ash.HashMap(c, a, sp, backend="delegate", device="cuda"),
                        "random_ops_delegate")


def test_delegate_backend(ash):
    G.replay_delegate(lambda c, a, sp, b: ash.HashMap(c, a, sp, backend=b, device="cuda"))


def test_growth_and_arity(ash):
    G.replay_growth(_mk(ash))


def test_voxel_downsample(ash):
    G.replay_voxel(lambda p, s: ash.voxel_downsample(p, s, device="cuda"))


def test_allocate_blocks(ash):
    G.replay_alloc_blocks(_mk(ash), lambda gm, c: ash.allocate_blocks(gm, c))


@pytest.mark.parametrize("seed", range(6))
def test_random_mixed_ops_vs_oracle(ash, O, seed):
    """Random op streams with heavy duplication and key reuse, compared step
    by step against the oracle (indices exact)."""
    rng = np.random.default_rng(1000 + seed)
    cap = int(rng.integers(50, 3000))
    arity = int(rng.choice([1, 2, 3, 4, 6]))
    specs = [np.float32, ((3,), np.int16)]
    g = ash.HashMap(cap, arity, specs, device="cuda")
    o = O.OracleMap(cap, arity, specs)
    span = int(rng.integers(2, 40))
    for step in range(40):
        op = rng.choice(["insert", "insert", "activate", "erase", "find", "rehash"])
        n = int(rng.integers(0, 4 * cap))
        keys = rng.integers(-span, span, size=(n, arity)).astype(np.int32)
        if op == "insert":
            v0 = rng.random(n, dtype=np.float32)
            v1 = rng.integers(-999, 999, size=(n, 3)).astype(np.int16)
            a, b = g.insert(keys, v0, v1), o.insert(keys, v0, v1)
        elif op == "activate":
            a, b = g.activate(keys), o.activate(keys)
        elif op == "find":
            a, b = g.find(keys), o.find(keys)
        elif op == "erase":
            G.eq(g.erase(keys), o.erase(keys), f"seed {seed} step {step} erase")
            continue
        else:
            c = max(o.size, 1) * int(rng.integers(1, 4))
            g.rehash(c)
            o.rehash(c)
            continue
        G.eq(a.indices, b.indices, f"seed {seed} step {step} {op} idx")
        G.eq(a.masks, b.masks, f"seed {seed} step {step} {op} mask")
        assert g.size == o.size and g.capacity == o.capacity
    G.eq(g.active_indices(), o.active_indices(), "active")
    G.bytes_eq(g.key_buffer, o.key_buffer, "keys")
    G.bytes_eq(g.value_buffer(0), o.value_buffer(0), "v0")
    G.bytes_eq(g.value_buffer(1), o.value_buffer(1), "v1")
    g.validate()


def test_heavy_duplication_winner_is_first(ash, O):
    """C4-like duplication (~900 copies per key): the lowest position wins."""
    rng = np.random.default_rng(7)
    pool = rng.integers(-2 ** 20, 2 ** 20, size=(1700, 3)).astype(np.int32)
    keys = pool[rng.integers(0, len(pool), size=1_536_000)]
    g = ash.HashMap(len(keys), 3, [np.int32], device="cuda")
    o = O.OracleMap(len(keys), 3, [np.int32])
    a, b = g.activate(keys), o.activate(keys)
    G.eq(a.indices, b.indices, "idx")
    G.eq(a.masks, b.masks, "mask")


def test_capacity_error_leaves_map_unchanged(ash):
    g = ash.HashMap(2, 3, [np.float32], auto_rehash=False, device="cuda")
    g.insert([[1, 1, 1], [2, 2, 2]], [1.0, 2.0])
    before = [to_np(x) for x in g.items_arrays()]
    with pytest.raises(ash.CapacityError):
        g.insert([[3, 3, 3], [4, 4, 4], [5, 5, 5]], [3.0, 4.0, 5.0])
    after = [to_np(x) for x in g.items_arrays()]
    assert all(np.array_equal(x, y) for x, y in zip(before, after))
    g.validate()
    # the rolled-back claims must not hide later inserts
    r = g.find([[3, 3, 3], [1, 1, 1]])
    assert to_np(r.masks).tolist() == [False, True]


def test_tombstone_churn_triggers_cleanup(ash):
    """insert/erase cycling (tests/test_hashmap.py:265-275) keeps working
    when tombstones would otherwise fill the table."""
    c = 32
    g = ash.HashMap(c, 3, [np.float32], auto_rehash=False, device="cuda")
    vals = np.ones((c, 1), np.float32)
    for it in range(300):
        keys = (np.arange(c * 3, dtype=np.int32) + 1000 * it).reshape(c, 3)
        assert bool(g.insert(keys, vals).masks.all())
        assert bool(g.erase(keys).all())
    assert g.size == 0
    g.validate()


def test_pipelined_host_batches_match_device_path(ash):
    """Pinned host batches take the chunked H2D/kernel/D2H pipeline; results
    (on the host) must equal the single-batch device path bit for bit."""
    import torch
    from paper_2110_00511_b200.workloads import int3_batch
    n = 5_000_000
    keys = torch.from_numpy(int3_batch(n, 0.3, seed=11)).pin_memory()
    vals = torch.rand((n, 2)).pin_memory()
    a = ash.HashMap(n, 3, [((2,), np.float32)], device="cuda")
    b = ash.HashMap(n, 3, [((2,), np.float32)], device="cuda")
    a.insert(keys[:1000].cuda(), vals[:1000].cuda())  # non-empty start: found vs new mix
    b.insert(keys[:1000].cuda(), vals[:1000].cuda())
    ra = a.insert(keys, vals)                      # pipelined (pinned, >= 1M rows)
    rb = b.insert(keys.cuda(), vals.cuda())        # one device batch
    assert not ra.indices.is_cuda and rb.indices.is_cuda
    assert torch.equal(ra.indices, rb.indices.cpu()) and torch.equal(ra.masks, rb.masks.cpu())
    assert a.size == b.size
    assert torch.equal(a.value_buffer(0), b.value_buffer(0)) and torch.equal(a._key_buf, b._key_buf)
    fa, fb = a.find(keys), b.find(keys.cuda())
    assert torch.equal(fa.indices, fb.indices.cpu()) and bool(fa.masks.all())
    # host (numpy) input -> host results
    r = a.find(keys[:10].numpy())
    assert not r.masks.is_cuda and bool(r.masks.all())


def test_ashl_snapshot_byte_identical_to_reference(ash, tmp_path):
    """serialize.py ASHL v1: the same op sequence gives the reference's exact
    snapshot bytes; the reference's snapshot loads back to the same content."""
    g = G.load("snapshot")
    m = ash.HashMap(64, 3, [((2,), np.float32), ((3,), np.uint8)], device="cuda")
    m.insert(g["keys"], g["v0"], g["v1"])
    m.erase(g["erase"])
    m.insert(g["k2"], g["k2v0"], g["k2v1"])
    path = tmp_path / "mine.ashl"
    m.save(path, metadata={"note": "golden"})
    assert path.read_bytes() == g["snap"].tobytes()
    ref = tmp_path / "ref.ashl"
    ref.write_bytes(g["snap"].tobytes())
    for backend in (None, "delegate"):
        loaded, meta = ash.HashMap.load(ref, backend=backend, device="cuda")
        assert meta == {"note": "golden"}
        assert loaded.capacity == 64 and loaded.size == m.size
        a, b = m.items_arrays(), loaded.items_arrays()
        # load re-inserts in ascending old-index order: rows are the same sequence
        assert all(np.array_equal(to_np(x), to_np(y)) for x, y in zip(a, b))
    bad = tmp_path / "junk.bin"
    bad.write_bytes(b"NOPE" + b"\0" * 64)
    with pytest.raises(ValueError, match="magic"):
        ash.HashMap.load(bad)


@pytest.mark.parametrize("arity", [3, 2, 1])
def test_dense_batches_vs_oracle(ash, O, arity):
    """Batches close to the capacity: indices exact against the oracle through
    duplicates, erase-made tombstones, activate of present keys, and keys
    with tens of thousands of copies."""
    rng = np.random.default_rng(77 + arity)
    cap = 120_000
    g = ash.HashMap(cap, arity, [np.float32], device="cuda")
    o = O.OracleMap(cap, arity, [np.float32])
    pool = rng.integers(-3000, 3000, size=(60_000, arity)).astype(np.int32)
    for step in range(4):
        keys = pool[rng.integers(0, len(pool), size=100_000)]
        if step == 2:  # two keys with 40k copies each
            keys[rng.permutation(100_000)[:80_000]] = pool[rng.integers(0, 2, size=80_000)]
        vals = rng.random((len(keys), 1), dtype=np.float32)
        a, b = g.insert(keys, vals), o.insert(keys, vals)
        G.eq(a.indices, b.indices, f"step {step} insert idx")
        G.eq(a.masks, b.masks, f"step {step} insert mask")
        G.eq(g.erase(keys[::3]), o.erase(keys[::3]), f"step {step} erase")
        a, b = g.activate(keys[::-1].copy()), o.activate(keys[::-1].copy())
        G.eq(a.indices, b.indices, f"step {step} activate idx")
        assert g.size == o.size
    G.eq(g.active_indices(), o.active_indices(), "active")
    G.bytes_eq(g.value_buffer(0), o.value_buffer(0), "values")
    g.validate()
