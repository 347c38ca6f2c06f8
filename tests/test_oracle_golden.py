"""Pin the CPU oracle against golden vectors recorded from the reference
itself (oracle/make_golden.py).  CPU only."""
import numpy as np
import pytest

import golden_replay as G
from oracle import ash_oracle as O


def make_oracle(cap, arity, specs):
    return O.OracleMap(cap, arity, specs)


def test_trace_appendix_a():
    G.replay_trace(make_oracle)


def test_c1_insert_find():
    G.replay_c1(make_oracle)


def test_bindings_parity_cases():
    G.replay_bindings(make_oracle)


def test_random_op_sequences():
    G.replay_random_ops(make_oracle)


def test_random_op_sequences_delegate():
    G.replay_random_ops(lambda c, a, sp: O.OracleMap(c, a, sp, backend="delegate"), "random_ops_delegate")


def test_delegate_backend():
    G.replay_delegate(lambda c, a, sp, b: O.OracleMap(c, a, sp, backend=b))


def test_growth_and_arity():
    G.replay_growth(make_oracle)


def test_voxel_downsample():
    G.replay_voxel(O.voxel_downsample)


def _cands(depth, intr, pose):
    cam = O.Camera(*intr[:4], int(intr[4]), int(intr[5]))
    return O.candidate_blocks(depth, cam, pose, 0.0058 * 8, 0.04)


def test_allocate_blocks_map_calls():
    def alloc(gm, coords):
        gi, local, _, _ = O.allocate_blocks_map_calls(gm, coords)
        return gi, local
    G.replay_alloc_blocks(make_oracle, alloc, _cands)


def test_lattice_hash_vectors():
    g = G.load("hash_dedup")
    for arity in (1, 2, 3, 4, 7):
        k = g[f"hash_keys_{arity}"]
        for n in (1, 37, 1000, 2 ** 20 + 7):
            G.eq(O.lattice_hash(k, n), g[f"hash_{arity}_{n}"], f"hash a{arity} n{n}")


def test_first_occurrence_vectors():
    g = G.load("hash_dedup")
    for name in ("fo_small", "fo_big", "fo_a1", "fo_a5"):
        G.eq(O.first_occurrence_mask(g[name + "_keys"]), g[name + "_mask"], name)


def test_gen_keys_vectors():
    g = G.load("hash_dedup")
    for cnt, rho, seed in ((1000, 0.5, 0), (5000, 0.1, 3), (777, 1.0, 9)):
        G.eq(O.gen_keys(cnt, rho, "int3", seed=seed), g[f"gen_{cnt}_{rho}_{seed}"], "gen_keys")


def test_heap_canonical_free_order():
    # index_heap tests: sorted free makes state a function of history
    h1, h2 = O.FreeList(8), O.FreeList(8)
    h1.allocate(5)
    h2.allocate(5)
    h1.free(np.array([4, 1, 3], np.int32))
    h2.free(np.array([3, 4, 1], np.int32))
    assert np.array_equal(h1.heap, h2.heap)
    with pytest.raises(O.HeapExhausted):
        h1.allocate(7)


def test_capacity_error_leaves_content():
    m = O.OracleMap(2, 3, [np.float32], auto_rehash=False)
    m.insert([[1, 1, 1], [2, 2, 2]], [1.0, 2.0])
    with pytest.raises(O.OracleCapacityError):
        m.insert([[3, 3, 3], [4, 4, 4], [5, 5, 5]], [3.0, 4.0, 5.0])
    assert m.size == 2
