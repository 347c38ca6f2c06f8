"""The semantics contract of DESIGN.md §2 as an executable spec: a
position-by-position dict model of the reference generic backend (SURVEY
App. A; hashmap.py:336-472, index_heap.py:14-55), written independently of
the oracle's vectorised chain walk, checked against the oracle on random op
sequences (hypothesis).  The oracle itself is pinned by reference-written
goldens (test_oracle_golden.py); this pins the contract the CUDA path is
tested against in words, one rule per line."""
import numpy as np
import pytest
from hypothesis import given, settings, strategies as st

from oracle.ash_oracle import OracleMap


class DictModel:
    def __init__(self, capacity):
        self._reset(capacity)

    def _reset(self, capacity):
        self.capacity = capacity
        self.heap = list(range(capacity))  # heap[top:] are free
        self.top = 0
        self.index = {}                    # present key -> buffer index
        self.rows = {}                     # buffer index -> key

    def _winners(self, keys):
        seen, win = set(), []
        for j, k in enumerate(keys):
            if k not in self.index and k not in seen:  # found[j] false, first in batch
                win.append(j)
            seen.add(k)
        return win

    def _rehash(self, capacity):
        # live rows in ascending old index become rows 0..size-1 (hashmap.py:326-332)
        live = [self.rows[i] for i in sorted(self.rows)]
        self._reset(capacity)
        for k in live:
            self._take(k)

    def _take(self, k):
        i = self.heap[self.top]
        self.top += 1
        self.index[k] = i
        self.rows[i] = k
        return i

    def insert(self, keys, assoc=False):
        while True:
            win = self._winners(keys)
            free = self.capacity - self.top
            if len(win) <= free:
                break
            cap = self.capacity
            while cap - len(self.index) < len(win):  # doubling (hashmap.py:311-324)
                cap *= 2
            self._rehash(cap)                        # then re-plan (hashmap.py:389-396)
        found = {j: self.index[k] for j, k in enumerate(keys) if k in self.index}
        idx, msk = [-1] * len(keys), [False] * len(keys)
        for j in win:                                # rank r takes heap[top + r]
            idx[j], msk[j] = self._take(keys[j]), True
        if assoc:                                    # activate: found positions too
            for j, i in found.items():
                idx[j], msk[j] = i, True
        return idx, msk

    def find(self, keys):
        idx = [self.index.get(k, -1) for k in keys]
        return idx, [i >= 0 for i in idx]

    def erase(self, keys):
        out, freed = [False] * len(keys), []
        for j, k in enumerate(keys):                 # first found occurrence per key
            if k in self.index:
                i = self.index.pop(k)
                del self.rows[i]
                freed.append(i)
                out[j] = True
        if freed:                                    # sorted, just below top (index_heap.py:38-47)
            self.top -= len(freed)
            self.heap[self.top:self.top + len(freed)] = sorted(freed)
        return out


OPS = st.lists(st.tuples(st.sampled_from(["insert", "insert", "activate", "find", "erase"]),
                         st.lists(st.integers(-6, 6), min_size=0, max_size=40)),
               min_size=1, max_size=25)


@settings(max_examples=150, deadline=None)
@given(ops=OPS, capacity=st.integers(1, 12))
def test_oracle_follows_the_dict_model(ops, capacity):
    o, m = OracleMap(capacity, 1), DictModel(capacity)
    for op, raw in ops:
        keys = np.asarray(raw, dtype=np.int32).reshape(-1, 1)
        tup = [int(k) for k in raw]
        if op == "erase":
            assert o.erase(keys).tolist() == m.erase(tup)
        else:
            r = getattr(o, op)(keys)
            idx, msk = (m.insert(tup, assoc=op == "activate") if op != "find" else m.find(tup))
            assert r.indices.tolist() == idx, op
            assert r.masks.tolist() == msk, op
        assert o.size == len(m.index) and o.capacity == m.capacity
        assert o.active_indices().tolist() == sorted(m.rows)
        assert o.heap.top == m.top and o.heap.heap.tolist() == m.heap


def test_model_appendix_a_rules():
    """The contract's corner cases, spelled out."""
    m = DictModel(4)
    assert m.insert([5, 5, 7]) == ([0, -1, 1], [True, False, True])  # first occurrence wins
    assert m.insert([7, 9]) == ([-1, 2], [False, True])               # present: masked, not re-indexed
    assert m.insert([9, 1], assoc=True) == ([2, 3], [True, True])      # activate reports found indices
    assert m.erase([7, 5, 7]) == [True, True, False]                   # one True per removed key
    assert m.heap == [0, 1, 0, 1] and m.top == 2                       # sorted frees below top
    assert m.insert([11, 12]) == ([0, 1], [True, True])                # lowest free index first
    assert m.insert([20, 21, 22]) == ([4, 5, 6], [True, True, True])   # grows 4 -> 8: live rows
    assert m.capacity == 8 and m.index == {11: 0, 12: 1, 9: 2, 1: 3, 20: 4, 21: 5, 22: 6}  # compacted by old index


@pytest.mark.parametrize("seed", range(3))
def test_model_matches_oracle_on_arity3_batches(seed):
    rng = np.random.default_rng(seed)
    o, m = OracleMap(64, 3), DictModel(64)
    for _ in range(12):
        keys = rng.integers(-3, 3, size=(int(rng.integers(0, 120)), 3)).astype(np.int32)
        tup = [tuple(int(x) for x in row) for row in keys]
        op = rng.choice(["insert", "activate", "erase", "find"])
        if op == "erase":
            assert o.erase(keys).tolist() == m.erase(tup)
            continue
        r = getattr(o, op)(keys)
        idx, msk = m.insert(tup, assoc=op == "activate") if op != "find" else m.find(tup)
        assert r.indices.tolist() == idx and r.masks.tolist() == msk
