"""Device-sized batches (ash_insert_dn / ash_find_dn) and the fused
dedup + activate sequences built on them (ash_allocate_blocks /
ash_allocate_frame): results identical to the host-sized calls and to the
oracle; the device capacity guard commits nothing when the new keys do not
fit (hashmap.py:389-396 raises before any change), and the Python layer then
falls back to the host-checked activate with doubling growth."""
import numpy as np
import pytest
import torch

import golden_replay as G

pytestmark = pytest.mark.gpu

BLOCK, TRUNC = 0.0058 * 8, 0.04


@pytest.fixture(scope="module")
def ash(cuda_ok):
    import paper_2110_00511_b200 as ash
    return ash


def _dn_insert(m, keys, vals, d_len, assoc=0):
    from paper_2110_00511_b200 import _lib
    n_max = keys.shape[0]
    d_n = torch.tensor([d_len], dtype=torch.int32, device="cuda")
    idx = torch.empty(n_max, dtype=torch.int32, device="cuda")
    msk = torch.empty(n_max, dtype=torch.uint8, device="cuda")
    m._ensure_scan(n_max)
    vptr = (_lib.c_void_p * 1)(vals.data_ptr()) if vals is not None else None
    _lib.call("ash_insert_dn", m._ptr(), keys.data_ptr(), n_max, d_n.data_ptr(), vptr, assoc,
              idx.data_ptr(), msk.data_ptr(), m._stream())
    flags = int(m._counters[_lib.CTR_FLAGS].item())
    m._size_known = False
    m._top_ub = m.capacity
    return idx[:d_len], msk[:d_len].view(torch.bool), flags


def test_insert_dn_equals_host_sized_insert(ash):
    from paper_2110_00511_b200 import _lib
    rng = np.random.default_rng(21)
    keys = torch.from_numpy(rng.integers(-300, 300, size=(300_000, 3)).astype(np.int32)).cuda()
    vals = torch.rand((300_000, 1), device="cuda")
    for d_len in (0, 1, 2047, 2048, 150_001, 300_000):
        a = ash.HashMap(400_000, 3, [np.float32], device="cuda")
        b = ash.HashMap(400_000, 3, [np.float32], device="cuda")
        ia, ma, flags = _dn_insert(a, keys, vals, d_len)
        assert flags & ~_lib.FLAG_SPEC == 0
        rb = b.insert(keys[:d_len], vals[:d_len])
        assert torch.equal(ia, rb.indices) and torch.equal(ma, rb.masks), d_len
        assert a.size == b.size
        assert torch.equal(a.value_buffer(0), b.value_buffer(0))
        q = keys[::3].contiguous()
        d_q = torch.tensor([q.shape[0] // 2], dtype=torch.int32, device="cuda")
        idx = torch.full((q.shape[0],), -7, dtype=torch.int32, device="cuda")
        msk = torch.zeros(q.shape[0], dtype=torch.uint8, device="cuda")
        _lib.call("ash_find_dn", a._ptr(), q.data_ptr(), q.shape[0], d_q.data_ptr(), idx.data_ptr(),
                  msk.data_ptr(), a._stream())
        h = q.shape[0] // 2
        fb = b.find(q[:h])
        assert torch.equal(idx[:h], fb.indices) and bool((idx[h:] == -7).all())
        a.validate()


def test_insert_dn_capacity_guard_commits_nothing(ash):
    from paper_2110_00511_b200 import _lib
    rng = np.random.default_rng(22)
    base = torch.from_numpy(rng.integers(-50, 50, size=(900, 3)).astype(np.int32)).cuda()
    m = ash.HashMap(1000, 3, [np.float32], device="cuda")
    r0 = m.insert(base, torch.rand((900, 1), device="cuda"))
    size0, keys0, vals0 = m.size, m.key_buffer.clone(), m.value_buffer(0).clone()
    act0 = m.active_indices()
    new = torch.from_numpy(rng.integers(1000, 2000, size=(5000, 3)).astype(np.int32)).cuda()
    idx, msk, flags = _dn_insert(m, new, torch.rand((5000, 1), device="cuda"), 5000)
    assert flags & (_lib.FLAG_CAPACITY | _lib.FLAG_TABLE_FULL)
    _lib.call("ash_insert_rollback", m._ptr(), 5000, idx.data_ptr(), m._stream())
    m._tombs_ub += 5000
    assert m.size == size0
    assert torch.equal(m.key_buffer, keys0) and torch.equal(m.value_buffer(0), vals0)
    assert torch.equal(m.active_indices(), act0)
    f = m.find(base)
    assert bool(f.masks.all()) and torch.equal(f.indices[r0.masks], r0.indices[r0.masks])
    assert not bool(m.find(new).masks.any())
    m.validate()


def test_fused_allocate_blocks_growth_fallback(ash):
    """A global map too small for the frame's blocks: the fused sequence's
    guard rejects the activate, the host path grows the map (doubling) and
    the indices equal the reference's (oracle with auto-rehash)."""
    from oracle import ash_oracle as O
    cam = O.scaled_camera(160, 120)
    depth = O.sphere_depth(cam)
    coords = O.candidate_blocks(depth, cam, np.eye(4), BLOCK, TRUNC)
    gm = ash.HashMap(16, 3, [((8, 8, 8, 2), np.float32)], device="cuda")
    og = O.OracleMap(16, 3, [((8, 8, 8, 2), np.float32)])
    gi, local = ash.allocate_blocks(gm, coords)
    gi_ref, _, _, _ = O.allocate_blocks_map_calls(og, coords)
    G.eq(gi, gi_ref, "gi after growth")
    assert gm.capacity == og.capacity and gm.size == og.size
    G.eq(gm.active_indices(), og.active_indices(), "active")
    G.bytes_eq(gm.key_buffer, og.key_buffer, "keys")
    # the frame path on the grown map: nothing new, same indices
    grid_gi, _ = ash.allocate_frame(gm, depth, cam, np.eye(4), BLOCK, TRUNC)
    G.eq(grid_gi, gi_ref, "frame path, existing blocks")
    gm.validate()


def test_fused_allocate_frames_sequence_matches_oracle(ash):
    """Ten posed frames through allocate_frame and allocate_blocks into two
    maps: indices, keys and active sets equal the oracle's map calls."""
    from oracle import ash_oracle as O
    cam = O.scaled_camera(320, 240)
    depth = O.plane_depth(cam, 1.0)
    g1 = ash.HashMap(3000, 3, [((8, 8, 8, 2), np.float32)], device="cuda")
    g2 = ash.HashMap(3000, 3, [((8, 8, 8, 2), np.float32)], device="cuda")
    og = O.OracleMap(3000, 3, [((8, 8, 8, 2), np.float32)])
    for f in range(10):
        pose = np.eye(4)
        pose[0, 3] = 0.05 * f
        pose[2, 3] = 0.01 * f
        coords = O.candidate_blocks(depth, cam, pose, BLOCK, TRUNC)
        gi_ref, _, _, _ = O.allocate_blocks_map_calls(og, coords)
        a, _ = ash.allocate_frame(g1, depth, cam, pose, BLOCK, TRUNC)
        b, _ = ash.allocate_blocks(g2, coords)
        G.eq(a, gi_ref, f"frame {f} allocate_frame")
        G.eq(b, gi_ref, f"frame {f} allocate_blocks")
    for gm in (g1, g2):
        assert gm.capacity == og.capacity and gm.size == og.size
        G.eq(gm.active_indices(), og.active_indices(), "active")
        G.bytes_eq(gm.key_buffer, og.key_buffer, "keys")
        gm.validate()


def test_fused_allocate_workspace_overflow_leaves_map_untouched(ash):
    """A frame with many more distinct blocks than the previous call's
    estimate overflows the workspace prefix: the global activate of that
    attempt takes 0 rows, the retry on the full table gives exact results."""
    from oracle import ash_oracle as O
    from paper_2110_00511_b200.blocks import unique_rows
    rng = np.random.default_rng(5)
    tiny = torch.from_numpy(rng.integers(0, 2, size=(50_000, 3)).astype(np.int32)).cuda()
    unique_rows(tiny)  # estimate = 8 distinct rows
    coords = rng.integers(-2 ** 20, 2 ** 20, size=(300_000, 3)).astype(np.int32)
    coords[1::5] = coords[::5][: len(coords[1::5])]
    gm = ash.HashMap(400_000, 3, device="cuda")
    og = O.OracleMap(400_000, 3)
    gi, _ = ash.allocate_blocks(gm, coords)
    gi_ref, _, _, _ = O.allocate_blocks_map_calls(og, coords)
    G.eq(gi, gi_ref, "gi")
    assert gm.size == og.size
    gm.validate()


def test_graph_replay_alternating_sequences(ash):
    """Two frames of different sizes alternate (each sequence is captured on
    its second occurrence and replayed after that, with the claim re-pointed
    at the frame's rows): every call equals the oracle's map calls."""
    from oracle import ash_oracle as O
    cams = [O.scaled_camera(160, 120), O.scaled_camera(200, 150)]
    frames = []
    for i, cam in enumerate(cams):
        depth = O.sphere_depth(cam) if i else O.plane_depth(cam, 1.0)
        for f in range(3):
            pose = np.eye(4)
            pose[0, 3] = 0.03 * f
            frames.append(O.candidate_blocks(depth, cam, pose, BLOCK, TRUNC))
    order = [0, 3, 1, 4, 2, 5, 0, 3, 1, 4, 2, 5]
    gm = ash.HashMap(20_000, 3, [((8, 8, 8, 2), np.float32)], device="cuda")
    og = O.OracleMap(20_000, 3, [((8, 8, 8, 2), np.float32)])
    for i in order:
        gi, _ = ash.allocate_blocks(gm, frames[i])
        gi_ref, _, _, _ = O.allocate_blocks_map_calls(og, frames[i])
        G.eq(gi, gi_ref, f"frame {i}")
    assert gm.size == og.size
    G.bytes_eq(gm.key_buffer, og.key_buffer, "keys")
    gm.validate()


def test_one_block_activate_refuses_long_batches(ash):
    """The fused sequence picks the one-block activate from the previous
    call's count; a batch with more distinct blocks than it takes (8192) is
    left untouched on the device and activated on the host path, exactly."""
    from oracle import ash_oracle as O
    from paper_2110_00511_b200.blocks import unique_rows
    rng = np.random.default_rng(8)
    unique_rows(torch.from_numpy(rng.integers(0, 3, size=(10_000, 3)).astype(np.int32)).cuda())  # estimate 27
    gm = ash.HashMap(100_000, 3, device="cuda")
    og = O.OracleMap(100_000, 3)
    for size, span in ((30_000, 40), (30_000, 5), (200_000, 60)):
        coords = rng.integers(-span, span, size=(size, 3)).astype(np.int32)
        gi, _ = ash.allocate_blocks(gm, coords)
        gi_ref, _, _, _ = O.allocate_blocks_map_calls(og, coords)
        G.eq(gi, gi_ref, f"{size}/{span}")
    assert gm.size == og.size
    G.eq(gm.active_indices(), og.active_indices(), "active")
    gm.validate()
