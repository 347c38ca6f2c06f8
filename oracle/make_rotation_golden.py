"""Golden digests of the REFERENCE's block candidates under general (non
axis-aligned) camera rotations.

Run in the build container (where /root/reference exists):

    python oracle/make_rotation_golden.py

``VoxelBlockGrid._candidate_blocks`` (pkg/src/spatialhash/tsdf/grid.py:98-125)
computes the world points as ``pts @ rot.T + trans`` with numpy's BLAS; the
rounding of that product decides a few boundary samples.  The device kernel
evaluates it as numpy's OpenBLAS dgemm kernel does on x86 (an FMA chain
over k = 0, 1, 2), so its candidates should equal the reference's
bit-for-bit.  This script records, for a few rotations, the SHA-256 of the
reference's candidate rows (int32, n x 3) and their count, written here by
the reference itself; ``tests/test_frame_gpu.py`` compares the kernel's
candidates with them (the GPU box's own numpy may use another BLAS kernel,
so the host oracle is not the reference there).
"""
from __future__ import annotations

import hashlib
import json
import sys
from pathlib import Path

import numpy as np

REF = Path("/root/reference/pkg/src")
ROOT = Path(__file__).resolve().parent.parent
OUT = ROOT / "tests" / "golden" / "frame_rotation_sha.json"

# (quaternion w, x, y, z; translation; shape): rotations about skewed axes
CASES = [
    ((0.9, 0.2, -0.3, 0.25), (0.1, 0.2, 0.3), "plane"),
    ((0.7, -0.4, 0.5, 0.3), (-0.05, 0.02, 0.15), "sphere"),
    ((0.95, 0.05, 0.1, -0.28), (0.3, -0.1, 0.0), "plane"),
]


def pose_of(q, t) -> np.ndarray:
    w, x, y, z = np.asarray(q, np.float64) / np.linalg.norm(q)
    pose = np.eye(4)
    pose[:3, :3] = [[1 - 2 * (y * y + z * z), 2 * (x * y - w * z), 2 * (x * z + w * y)],
                    [2 * (x * y + w * z), 1 - 2 * (x * x + z * z), 2 * (y * z - w * x)],
                    [2 * (x * z - w * y), 2 * (y * z + w * x), 1 - 2 * (x * x + y * y)]]
    pose[:3, 3] = t
    return pose


def main() -> None:
    sys.path.insert(0, str(REF))
    from spatialhash.tsdf import TsdfConfig, VoxelBlockGrid
    from spatialhash.tsdf.synthetic import plane_depth, sphere_depth
    from spatialhash.tsdf.types import Frame, Intrinsics

    w, h = 320, 240
    intr = Intrinsics(fx=250.0, fy=250.0, cx=(w - 1) / 2, cy=(h - 1) / 2, width=w, height=h)
    cfg = TsdfConfig(0.0058, 8, 0.04)
    out = {"intrinsics": [intr.fx, intr.fy, intr.cx, intr.cy, w, h], "voxel": 0.0058, "block_resolution": 8,
           "trunc": 0.04, "cases": []}
    for q, t, shape in CASES:
        depth = plane_depth(intr, 1.2) if shape == "plane" else sphere_depth(intr, (0.0, 0.0, 1.0), 0.3)
        pose = pose_of(q, t)
        grid = VoxelBlockGrid(cfg, capacity=1000)
        coords = np.ascontiguousarray(grid._candidate_blocks(Frame(depth.copy(), intr, pose)), dtype=np.int32)
        out["cases"].append({"quaternion": list(q), "translation": list(t), "shape": shape,
                             "pose": pose.tolist(), "count": int(len(coords)),
                             "sha256": hashlib.sha256(coords.tobytes()).hexdigest()})
        print(shape, q, len(coords))
    OUT.write_text(json.dumps(out, indent=1))
    print("wrote", OUT)


if __name__ == "__main__":
    main()
