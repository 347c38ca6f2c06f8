"""Fused frame allocation: block candidates generated on
the device from the depth image (tsdf/grid.py:98-125, block_of :24-27), the
fused dedup (local activate, grid.py:140-142) and allocate_frame
(grid.py:127-150) against the reference's own outputs (golden
alloc_blocks.npz, written by the reference) and the oracle."""
from types import SimpleNamespace

import numpy as np
import pytest

import golden_replay as G

pytestmark = pytest.mark.gpu

BLOCK, TRUNC = 0.0058 * 8, 0.04


@pytest.fixture(scope="module")
def ash(cuda_ok):
    import paper_2110_00511_b200 as ash
    return ash


def _intr(v):
    fx, fy, cx, cy, w, h = v
    return SimpleNamespace(fx=fx, fy=fy, cx=cx, cy=cy, width=int(w), height=int(h))


def _first_occurrence_rows(coords):
    _, first = np.unique(coords, axis=0, return_index=True)
    return coords[np.sort(first)]


def test_golden_frames_candidates_and_allocation(ash):
    g = G.load("alloc_blocks")
    intr = _intr(g["intr"])
    for shape in ("plane", "sphere"):
        gm = ash.HashMap(5000, 3, [((8, 8, 8, 2), np.float32)], device="cuda")
        depth = g[f"{shape}_depth"]
        for f in range(3):
            p = f"{shape}_f{f}_"
            coords = g[p + "coords"]
            cand = ash.frame_candidates(depth, intr, g[p + "pose"], BLOCK, TRUNC, device="cuda")
            G.eq(cand, coords, f"{p} candidates")
            blocks = ash.frame_blocks(depth, intr, g[p + "pose"], BLOCK, TRUNC, device="cuda")
            G.eq(blocks, _first_occurrence_rows(coords), f"{p} distinct blocks")
            gi, local = ash.allocate_frame(gm, depth, intr, g[p + "pose"], BLOCK, TRUNC)
            G.eq(gi, g[p + "gi"], f"{p} gi")
            G.eq(local.find(coords).indices, g[p + "local_find_idx"], f"{p} local idx")
            G.bytes_eq(local.value_buffer(0), g[p + "local_values"], f"{p} local values")
        G.bytes_eq(gm.key_buffer, g[f"{shape}_global_keys"], f"{shape} global keys")
        G.eq(gm.active_indices(), g[f"{shape}_global_active"], f"{shape} global active")


@pytest.mark.parametrize("shape", ["plane", "sphere"])
def test_full_frame_matches_oracle(ash, shape):
    from oracle import ash_oracle as O
    cam = O.scaled_camera(640, 480)
    depth = O.plane_depth(cam, 1.0) if shape == "plane" else O.sphere_depth(cam)
    pose = np.eye(4)
    pose[:3, 3] = [0.02, -0.01, 0.005]
    want = O.candidate_blocks(depth, cam, pose, BLOCK, TRUNC)
    got = ash.frame_candidates(depth, cam, pose, BLOCK, TRUNC, device="cuda")
    G.eq(got, want, "candidates")
    G.eq(ash.frame_blocks(depth, cam, pose, BLOCK, TRUNC, device="cuda"), _first_occurrence_rows(want),
         "blocks")
    grid = ash.BlockGrid(8, capacity=100_000, device="cuda")
    gi = grid.allocate_frame(depth, cam, pose)
    og = O.OracleMap(100_000, 3, [((8, 8, 8, 2), np.float32)])
    gi_ref, _, _, _ = O.allocate_blocks_map_calls(og, want)
    G.eq(gi, gi_ref, "gi")


def test_axis_aligned_rotation_exact_and_neighbor_mode(ash):
    from oracle import ash_oracle as O
    cam = O.scaled_camera(320, 240)
    depth = O.sphere_depth(cam, (0.05, 0.0, 1.0), 0.4)
    depth[::7, ::5] = np.nan  # invalid samples: NaN fails every valid_mask comparison
    depth[1::9, ::3] = 3.5    # beyond depth_max
    pose = np.zeros((4, 4))
    pose[0, 1], pose[1, 2], pose[2, 0], pose[3, 3] = 1.0, -1.0, 1.0, 1.0  # axis permutation
    pose[:3, 3] = [0.3, 0.1, -0.2]
    G.eq(ash.frame_candidates(depth, cam, pose, BLOCK, TRUNC, device="cuda"),
         O.candidate_blocks(depth, cam, pose, BLOCK, TRUNC), "ray candidates")
    # neighbor mode (tsdf/grid.py:108-113): surface block + lattice_offsets(1)
    ok = (depth > 0) & (depth >= 0.2) & (depth <= 3.0)
    v, u = np.nonzero(ok)
    surf = cam.unproject(u, v, 1.0) * depth[v, u][:, None]
    world = surf @ pose[:3, :3].T + pose[:3, 3]
    blocks = np.floor(world / BLOCK).astype(np.int32)
    offs = np.array([(a, b, c) for a in (-1, 0, 1) for b in (-1, 0, 1) for c in (-1, 0, 1)], np.int32)
    want = (blocks[:, None, :] + offs[None]).reshape(-1, 3)
    got = ash.frame_candidates(depth, cam, pose, BLOCK, TRUNC, allocation="neighbor", device="cuda")
    G.eq(got, want, "neighbor candidates")
    G.eq(ash.frame_blocks(depth, cam, pose, BLOCK, TRUNC, allocation="neighbor", device="cuda"),
         _first_occurrence_rows(want), "neighbor blocks")


def test_general_rotation_follows_blas_fma_order(ash):
    """A general rotation: the kernel evaluates the pose product as an FMA
    chain (numpy's OpenBLAS dgemm on x86).  Bit-exact where the host BLAS uses
    that kernel; a different host kernel may round a boundary sample the
    other way, so this bounds the disagreement instead."""
    from oracle import ash_oracle as O
    cam = O.scaled_camera(320, 240)
    depth = O.plane_depth(cam, 1.2)
    q = np.array([0.9, 0.2, -0.3, 0.25])
    w, x, y, z = q / np.linalg.norm(q)
    pose = np.eye(4)
    pose[:3, :3] = [[1 - 2 * (y * y + z * z), 2 * (x * y - w * z), 2 * (x * z + w * y)],
                    [2 * (x * y + w * z), 1 - 2 * (x * x + z * z), 2 * (y * z - w * x)],
                    [2 * (x * z - w * y), 2 * (y * z + w * x), 1 - 2 * (x * x + y * y)]]
    pose[:3, 3] = [0.1, 0.2, 0.3]
    want = O.candidate_blocks(depth, cam, pose, BLOCK, TRUNC)
    got = G.to_np(ash.frame_candidates(depth, cam, pose, BLOCK, TRUNC, device="cuda"))
    assert got.shape == want.shape
    assert np.count_nonzero((got != want).any(axis=1)) <= len(want) // 10_000


def test_empty_and_invalid_frames(ash):
    cam = SimpleNamespace(fx=100.0, fy=100.0, cx=15.5, cy=11.5, width=32, height=24)
    zero = np.zeros((24, 32))
    assert ash.frame_blocks(zero, cam, np.eye(4), BLOCK, TRUNC, device="cuda").shape == (0, 3)
    gm = ash.HashMap(16, 3, device="cuda")
    gi, local = ash.allocate_frame(gm, zero, cam, np.eye(4), BLOCK, TRUNC)
    assert gi.numel() == 0 and local is None and gm.size == 0
    with pytest.raises(ValueError):
        ash.frame_blocks(np.ones((10, 10)), cam, np.eye(4), BLOCK, TRUNC, device="cuda")
    with pytest.raises(ValueError):
        ash.frame_blocks(np.ones((24, 32)), cam, np.eye(4), BLOCK, TRUNC, allocation="cone",
                         device="cuda")


def test_unique_rows_and_workspace_overflow_retry(ash):
    """ash_unique_rows == first occurrences; a call after a much smaller one
    overflows the estimate-sized workspace prefix (bounded probe) and must be
    retried on the full table — results stay exact either way."""
    import torch
    from paper_2110_00511_b200.blocks import unique_rows
    rng = np.random.default_rng(12)
    small = torch.from_numpy(rng.integers(-3, 3, size=(100_000, 3)).astype(np.int32)).cuda()
    got = unique_rows(small)
    G.eq(got, _first_occurrence_rows(small.cpu().numpy()), "small")
    big = rng.integers(-2 ** 30, 2 ** 30, size=(400_000, 3)).astype(np.int32)  # all distinct
    big[::7] = big[3]  # a few repeats
    got = unique_rows(torch.from_numpy(big).cuda())
    G.eq(got, _first_occurrence_rows(big), "big after small (retried)")
    got = unique_rows(small)
    G.eq(got, _first_occurrence_rows(small.cpu().numpy()), "small again")


def test_general_rotations_match_reference_digests(ash):
    """General rotations against the reference itself: digests of
    VoxelBlockGrid._candidate_blocks written by the reference in the build
    container (oracle/make_rotation_golden.py), where numpy's OpenBLAS
    evaluates the pose product as the kernel does (an FMA chain): bit-exact,
    independent of the GPU box's own BLAS."""
    import hashlib
    import json
    from pathlib import Path
    from oracle import ash_oracle as O
    g = json.loads((Path(__file__).parent / "golden" / "frame_rotation_sha.json").read_text())
    cam = O.scaled_camera(320, 240)
    block = g["voxel"] * g["block_resolution"]
    for case in g["cases"]:
        depth = O.plane_depth(cam, 1.2) if case["shape"] == "plane" else O.sphere_depth(cam)
        pose = np.array(case["pose"])
        got = np.ascontiguousarray(G.to_np(ash.frame_candidates(depth, cam, pose, block, g["trunc"],
                                                                device="cuda")), dtype=np.int32)
        assert len(got) == case["count"], case["quaternion"]
        assert hashlib.sha256(got.tobytes()).hexdigest() == case["sha256"], case["quaternion"]


@pytest.mark.parametrize("w,h", [(37, 23), (61, 7), (5, 3)])
def test_ragged_frames_distinct_blocks_match_oracle(ash, w, h):
    """Image sizes whose candidate counts end inside a claim block (the
    per-block pixel-ray table of the frame claim over a partial block, a
    block spanning two image rows): frame_blocks and allocate_frame equal the
    first-occurrence rows of the oracle's candidates, translated pose."""
    from oracle import ash_oracle as O
    from paper_2110_00511_b200.blocks import allocate_frame
    cam = O.Camera(fx=30.0, fy=31.0, cx=(w - 1) / 2, cy=(h - 1) / 2, width=w, height=h)
    pose = np.eye(4)
    pose[:3, 3] = [0.013, -0.021, 0.007]
    for depth in (O.plane_depth(cam, 0.9), O.sphere_depth(cam, radius=0.5)):
        coords = O.candidate_blocks(depth, cam, pose, BLOCK, TRUNC)
        want = _first_occurrence_rows(coords) if len(coords) else coords.reshape(0, 3)
        G.eq(ash.frame_blocks(depth, cam, pose, BLOCK, TRUNC, device="cuda"), want, f"{w}x{h} blocks")
        gm = ash.HashMap(4096, 3, [np.float32], device="cuda")
        gi, _ = allocate_frame(gm, depth, cam, pose, BLOCK, TRUNC)
        assert gm.size == len(want)
        G.eq(gi, G.to_np(gm.find(want).indices), f"{w}x{h} gi")
