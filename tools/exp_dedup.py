"""configs[2] / configs[3] dedup-select paths on the GPU box: per-call device
time (CUDA events) of voxel_downsample (20M sphere points), allocate_blocks
(given 1.536M candidates) and BlockGrid.allocate_frame (from the depth image).

  python tools/exp_dedup.py [c3|c4|c4f|all] [reps]

Run under `ncu --metrics gpu__time_duration.sum` for the launch list, or
`ncu --set full -k regex:k_voxel_claim` for one capture."""
import statistics
import sys

sys.path.insert(0, ".")
import numpy as np
import torch

import paper_2110_00511_b200 as ash
from oracle import ash_oracle as O
from paper_2110_00511_b200.workloads import sphere_points

dev = torch.device("cuda:0")
what = sys.argv[1] if len(sys.argv) > 1 else "all"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 6
stream = torch.cuda.current_stream(dev)


def timed(fn):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(stream)
    r = fn()
    b.record(stream)
    torch.cuda.synchronize()
    return a.elapsed_time(b), r


if what in ("c3", "all"):
    pts = torch.from_numpy(sphere_points(20_000_000, seed=0)).to(dev)
    ts = []
    for i in range(reps):
        t, (c, s) = timed(lambda: ash.voxel_downsample(pts, 0.005, device=dev))
        ts.append(t)
    print("c3 voxelize ms", [round(x, 3) for x in ts], "median", round(statistics.median(ts[1:]), 4),
          "voxels", c.shape[0], flush=True)

if what in ("c4", "c4f", "all"):
    cam = O.scaled_camera(640, 480)
    depth = O.plane_depth(cam, 1.0)
    poses = []
    for f in range(10):
        p = np.eye(4)
        p[0, 3] = 0.02 * f
        poses.append(p)
    if what in ("c4", "all"):
        frames = [torch.from_numpy(O.candidate_blocks(depth, cam, p, 0.0058 * 8, 0.04)).to(dev) for p in poses]
        gm = ash.HashMap(100_000, 3, [((8, 8, 8, 2), np.float32)], device=dev)
        ts = []
        for rep in range(2):
            gm.clear()
            for c in frames:
                t, _ = timed(lambda: ash.allocate_blocks(gm, c))
                if rep:
                    ts.append(t)
        print("c4 allocate_blocks ms/frame", [round(x, 3) for x in ts], "median", round(statistics.median(ts), 4),
              "blocks", gm.size, flush=True)
    if what in ("c4f", "all"):
        depth_d = torch.from_numpy(depth).to(dev)
        grid = ash.BlockGrid(8, capacity=100_000, device=dev)
        ts = []
        for rep in range(2):
            grid.global_map.clear()
            for p in poses:
                t, _ = timed(lambda: grid.allocate_frame(depth_d, cam, p))
                if rep:
                    ts.append(t)
        print("c4 allocate_frame ms/frame", [round(x, 3) for x in ts], "median", round(statistics.median(ts), 4),
              "blocks", grid.block_count, flush=True)
