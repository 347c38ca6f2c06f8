"""Parity at BASELINE.json's full sizes through size-independent properties.

The oracle would take minutes here, so these checks use an independent
torch checker: sort-based unique + first occurrence (scatter_reduce amin
over positions), which must agree exactly with the map's masks/indices."""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ash(cuda_ok):
    import paper_2110_00511_b200 as ash
    return ash


def first_occurrence(keys: torch.Tensor):
    """(inverse group id per row, first position per group, n_groups)."""
    _, inv = torch.unique(keys, dim=0, return_inverse=True)
    g = int(inv.max().item()) + 1 if inv.numel() else 0
    pos = torch.arange(keys.shape[0], device=keys.device)
    first = torch.full((g,), keys.shape[0], dtype=torch.int64, device=keys.device)
    first.scatter_reduce_(0, inv, pos, reduce="amin")
    return inv, first, g


@pytest.mark.parametrize("rho", [0.1, 0.5, 1.0])
def test_c2_10m_insert_find_erase(ash, rho):
    from paper_2110_00511_b200.workloads import int3_batch
    n = 10_000_000
    keys = torch.from_numpy(int3_batch(n, rho, seed=7)).cuda()
    vals = torch.rand((n, 8), device="cuda")
    m = ash.HashMap(n, 3, [((8,), np.float32)], device="cuda")
    r = m.insert(keys, vals)
    inv, first, g = first_occurrence(keys)
    assert g == int(np.ceil(rho * n)) == m.size
    want = torch.zeros(n, dtype=torch.bool, device="cuda")
    want[first] = True
    assert torch.equal(r.masks, want)
    # fresh heap: winner of rank r gets index r (hashmap.py:397 with heap = arange)
    assert torch.equal(r.indices[r.masks], torch.arange(g, dtype=torch.int32, device="cuda"))
    assert torch.equal(r.indices[~r.masks], torch.full((n - g,), -1, dtype=torch.int32, device="cuda"))
    idx = r.indices[r.masks].long()
    assert torch.equal(m.key_buffer[idx], keys[r.masks])
    assert torch.equal(m.value_buffer(0)[idx], vals[r.masks])
    f = m.find(keys)
    assert bool(f.masks.all())
    # every position finds its key's winner index
    winner_idx = torch.empty(g, dtype=torch.int32, device="cuda")
    winner_idx[inv[first]] = r.indices[first]
    assert torch.equal(f.indices, winner_idx[inv])
    # activate: all found, same indices; size unchanged
    a = m.activate(keys)
    assert bool(a.masks.all()) and torch.equal(a.indices, f.indices) and m.size == g
    # erase the keys of even groups: exactly one mask per key, at its first occurrence
    even = (inv % 2 == 0)
    ek = keys[even]
    e = m.erase(ek)
    e_inv, e_first, e_g = first_occurrence(ek)
    want_e = torch.zeros(ek.shape[0], dtype=torch.bool, device="cuda")
    want_e[e_first] = True
    assert torch.equal(e, want_e) and m.size == g - e_g
    # freed indices return to the heap below top, ascending (index_heap.py:38-47)
    top = m.size
    freed = m._heap_buf[top:top + e_g]
    assert torch.equal(freed, torch.sort(r.indices[first][(inv[first] % 2) == 0]).values)
    f2 = m.find(keys)
    assert torch.equal(f2.masks, ~even)
    # re-insert: the freed indices are reused in ascending order
    r2 = m.insert(ek, vals[even])
    assert torch.equal(r2.masks, want_e)
    assert torch.equal(r2.indices[r2.masks], freed)
    m.validate()


def test_c3_voxelize_20m_sphere(ash):
    from paper_2110_00511_b200.workloads import sphere_points
    pts = torch.from_numpy(sphere_points(20_000_000, seed=0)).cuda()
    coords, sel = ash.voxel_downsample(pts, 0.005, device="cuda")
    q = ash.quantize(pts, 0.005, device="cuda")
    # quantization is float64 floor(p / s): spot-check against numpy on a sample
    smp = torch.randint(0, pts.shape[0], (200_000,), device="cuda")
    ref = np.floor(pts[smp].cpu().numpy() / 0.005).astype(np.int32)
    assert np.array_equal(q[smp].cpu().numpy(), ref)
    inv, first, g = first_occurrence(q)
    assert coords.shape[0] == g == 702_116  # reference result at C3
    assert torch.equal(sel, torch.sort(first).values)
    assert torch.equal(coords, q[sel])


def test_c4_allocate_blocks_full_frame(ash):
    from oracle import ash_oracle as O
    cam = O.scaled_camera(640, 480)
    depth = O.plane_depth(cam, 1.0)
    coords = O.candidate_blocks(depth, cam, np.eye(4), 0.0058 * 8, 0.04)
    assert len(coords) == 1_536_000
    og = O.OracleMap(100_000, 3, [((8, 8, 8, 2), np.float32)])
    gi_ref, local_ref, li, lmask = O.allocate_blocks_map_calls(og, coords)
    gm = ash.HashMap(100_000, 3, [((8, 8, 8, 2), np.float32)], device="cuda")
    gi, local = ash.allocate_blocks(gm, coords)
    assert np.array_equal(gi.cpu().numpy(), gi_ref)
    assert len(gi_ref) == 1_836  # fx = fy = 500 (cli.py:125-130 scaling of the 320-wide intrinsics)
    assert np.array_equal(local.find(coords).indices.cpu().numpy(), local_ref.find(coords).indices)
    assert local.value_buffer(0).cpu().numpy().tobytes() == local_ref.value_buffer(0).tobytes()
