"""Speculative pending states (k_claim, ASH_FLAG_SPEC).

While the index heap is the identity above its top, a claim marks its slots
top + position instead of PENDING | position, and a batch whose positions
all win is final after the claim (no slot-state stores, no table sweep).
Every op sequence must give results identical to the PENDING | position
encoding (ASH_SPEC=0, read per call) and to the oracle (hashmap.py:376-420
insert, 422-438 find, 440-466 erase)."""
import contextlib
import os

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


@contextlib.contextmanager
def spec(on):
    old = os.environ.get("ASH_SPEC")
    os.environ["ASH_SPEC"] = "1" if on else "0"
    try:
        yield
    finally:
        if old is None:
            del os.environ["ASH_SPEC"]
        else:
            os.environ["ASH_SPEC"] = old


def _state(m):
    return (m.key_buffer.clone(), m.value_buffer(0).clone() if m._value_bufs else None,
            m.active_indices().clone(), m.size)


def _run(ash, on, ops, capacity, arity, width=1):
    """Apply ops to a fresh map; return every result and the final state."""
    out = []
    with spec(on):
        m = ash.HashMap(capacity, arity, [((width,), np.float32)], device="cuda")
        for op, keys, vals in ops:
            if op == "insert":
                r = m.insert(keys, vals)
                out += [r.indices.clone(), r.masks.clone()]
            elif op == "activate":
                r = m.activate(keys)
                out += [r.indices.clone(), r.masks.clone()]
            elif op == "erase":
                out.append(m.erase(keys).clone())
            f = m.find(keys)
            out += [f.indices.clone(), f.masks.clone()]
        m.validate()
        return out, _state(m), m


def _assert_same(a, b, values=True):
    ra, sa, _ = a
    rb, sb, _ = b
    assert len(ra) == len(rb)
    for i, (x, y) in enumerate(zip(ra, rb)):
        assert torch.equal(x, y), f"result {i}"
    assert torch.equal(sa[0], sb[0]) and torch.equal(sa[2], sb[2]) and sa[3] == sb[3]
    if values and sa[1] is not None:
        assert torch.equal(sa[1], sb[1])


def _keys(rng, n, lo, hi, arity=3):
    return torch.from_numpy(rng.integers(lo, hi, size=(n, arity)).astype(np.int32)).cuda()


def test_all_new_distinct_batches_match(ash):
    """Distinct new keys (every position wins: states final after the
    claim), large enough for the sweep threshold, then small ones."""
    rng = np.random.default_rng(40)
    base = np.unique(rng.integers(-10 ** 6, 10 ** 6, size=(1_300_000, 3)).astype(np.int32), axis=0)
    base = base[rng.permutation(len(base))]
    big, small = torch.from_numpy(base[:1_000_000]).cuda(), torch.from_numpy(base[1_000_000:1_001_000]).cuda()
    ops = [("insert", big, torch.rand((big.shape[0], 1), device="cuda")),
           ("insert", small, torch.rand((small.shape[0], 1), device="cuda"))]
    a = _run(ash, True, ops, 1_200_000, 3)
    b = _run(ash, False, ops, 1_200_000, 3)
    _assert_same(a, b)
    # indices are exactly top + position for all-new batches (hashmap.py:403-409)
    assert torch.equal(a[0][0], torch.arange(1_000_000, dtype=torch.int32, device="cuda"))
    assert torch.equal(a[0][4], torch.arange(1_000_000, 1_001_000, dtype=torch.int32, device="cuda"))


@pytest.mark.parametrize("arity", [1, 2, 3])
def test_mixed_duplicates_and_present_keys_match_oracle(ash, arity):
    from oracle.ash_oracle import OracleMap
    rng = np.random.default_rng(41 + arity)
    k1 = _keys(rng, 400_000, -400, 400, arity)  # heavy duplication
    k2 = _keys(rng, 300_000, -900, 900, arity)  # part present, part new
    k3 = torch.cat([k1[:1000], _keys(rng, 200_000, 10 ** 5, 10 ** 6, arity)])  # mostly new
    ops = [("insert", k, torch.rand((k.shape[0], 1), device="cuda")) for k in (k1, k2, k3)]
    a = _run(ash, True, ops, 1_500_000, arity)
    b = _run(ash, False, ops, 1_500_000, arity)
    _assert_same(a, b)
    o = OracleMap(1_500_000, arity, [((1,), np.float32)])
    i = 0
    for _, keys, vals in ops:
        ri, rm = o.insert(keys.cpu().numpy(), vals.cpu().numpy())
        assert np.array_equal(a[0][i].cpu().numpy()[rm], ri[rm]) and np.array_equal(a[0][i + 1].cpu().numpy(), rm)
        i += 4
    assert a[1][3] == o.size


def test_after_erase_heap_not_identity(ash):
    """An erase frees indices below top: the next claims must not speculate
    (indices come from the heap), and results still match."""
    rng = np.random.default_rng(44)
    k1 = _keys(rng, 500_000, -10 ** 5, 10 ** 5)
    k2 = _keys(rng, 500_000, -10 ** 5, 10 ** 5)
    k3 = _keys(rng, 500_000, -2 * 10 ** 5, 2 * 10 ** 5)
    v = torch.rand((500_000, 1), device="cuda")
    ops = [("insert", k1, v), ("erase", k1[::3].contiguous(), None), ("insert", k2, v), ("insert", k3, v),
           ("activate", k1, None)]
    a = _run(ash, True, ops, 2_000_000, 3)
    b = _run(ash, False, ops, 2_000_000, 3)
    _assert_same(a, b, values=False)  # activate leaves value rows as they were
    act = a[1][2].long()
    _, _, ma = a
    _, _, mb = b
    keep = torch.ones(ma.capacity, dtype=torch.bool, device="cuda")
    r_act = a[0][-4]  # the activate's indices
    keep[r_act.long()] = False
    keep = keep[act]
    assert torch.equal(ma.value_buffer(0)[act][keep], mb.value_buffer(0)[act][keep])


def test_spec_claim_with_deferred_commit_sweeps_at_once(ash):
    """ash_insert_claim (speculative) followed by ash_insert_commit_lazy: the
    finds cannot resolve top + pos states, so the commit sweeps them at
    once; ash_settle is then a no-op.  Same results as the eager insert."""
    from paper_2110_00511_b200 import _lib
    rng = np.random.default_rng(45)
    keys = _keys(rng, 600_000, -200, 200)
    keys[::7] = _keys(rng, keys[::7].shape[0], 10 ** 6, 2 * 10 ** 6)
    vals = torch.rand((600_000, 1), device="cuda")
    with spec(True):
        ref = ash.HashMap(700_000, 3, [np.float32], device="cuda")
        r_ref = ref.insert(keys, vals)
        f_ref = ref.find(keys)
        m = ash.HashMap(700_000, 3, [np.float32], device="cuda")
        n = keys.shape[0]
        idx = torch.empty(n, dtype=torch.int32, device="cuda")
        msk = torch.empty(n, dtype=torch.uint8, device="cuda")
        m._ensure_scan(n)
        assert m._rank_words is not None
        vptr = (_lib.c_void_p * 1)(vals.data_ptr())
        s = m._stream()
        _lib.call("ash_insert_claim", m._ptr(), keys.data_ptr(), n, idx.data_ptr(), msk.data_ptr(), s)
        assert int(m._counters[_lib.CTR_FLAGS].item()) & _lib.FLAG_SPEC
        _lib.call("ash_insert_count", m._ptr(), n, idx.data_ptr(), msk.data_ptr(), s)
        _lib.call("ash_insert_commit_lazy", m._ptr(), keys.data_ptr(), n, vptr, 0, idx.data_ptr(), msk.data_ptr(), s)
        m._size_known = False
        m._top_ub = m.capacity
        assert torch.equal(idx, r_ref.indices) and torch.equal(msk.view(torch.bool), r_ref.masks)
        f = m.find(keys)
        assert torch.equal(f.indices, f_ref.indices) and torch.equal(f.masks, f_ref.masks)
        before = m._slots.clone()
        _lib.call("ash_settle", m._ptr(), s)
        assert torch.equal(m._slots, before)  # nothing was left pending
        st = before.view(-1, 4)[:, 3]
        assert bool(((st >= 0) & (st < m.size) | (st == -1) | (st == -2)).all())
        m.validate()
