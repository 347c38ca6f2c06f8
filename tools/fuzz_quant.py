"""Randomized voxel_downsample against the oracle at the points where the
cloud claim's reciprocal-multiply quantize could round to the wrong side
(GPU box): random cells (log-uniform 1e-6 .. 1e4 and awkward decimals),
points at integer multiples of the cell and 1-4 ulps around them, magnitudes
up to and past 2^30 cells (the fast path's range limit), zeros, subnormals,
float32 and float64 clouds.  Exact coords and selection indices.
    python tools/fuzz_quant.py FIRST_SEED END_SEED"""
import os
import sys

sys.path.insert(0, os.getcwd())
sys.path.insert(0, os.path.join(os.getcwd(), "tests"))
import numpy as np
import torch

import golden_replay as G
import paper_2110_00511_b200 as ash
from oracle import ash_oracle as O

fails = 0
for seed in range(int(sys.argv[1]), int(sys.argv[2])):
    rng = np.random.default_rng(seed)
    try:
        cell = float(rng.choice([10 ** rng.uniform(-6, 4), 0.1, 0.005, 1 / 3, 0.0058 * 8, 7.3e-4, 1.1]))
        n = int(rng.choice([64, 1000, 50_000, 300_000]))
        top = float(rng.choice([100, 1e4, 2.0 ** 29, 2.0 ** 30 + 5, 2.0 ** 31 - 3]))
        k = np.floor(rng.uniform(-top, top, size=n))
        pts = k * cell
        steps = rng.integers(-4, 5, size=n)
        for s in range(1, 5):  # move each point 0-4 ulps up or down
            up, dn = steps >= s, steps <= -s
            pts[up] = np.nextafter(pts[up], np.inf)
            pts[dn] = np.nextafter(pts[dn], -np.inf)
        free = rng.random(n) < 0.3
        pts[free] = rng.uniform(-top, top, size=int(free.sum())) * cell
        special = np.array([0.0, -0.0, 5e-324, -5e-324, 1e-310, -1e-310, cell, -cell])
        pts[: len(special)] = special[: n]
        pts = pts[np.abs(pts / cell) < 2.0 ** 31 - 2]
        m = len(pts) // 3 * 3
        cloud = pts[:m].reshape(-1, 3)
        if rng.random() < 0.3:
            cloud = cloud.astype(np.float32)
            cloud = cloud[np.all(np.abs(cloud.astype(np.float64) / cell) < 2.0 ** 31 - 2, axis=1)]
        cloud = cloud[rng.permutation(len(cloud))]
        c, s = ash.voxel_downsample(torch.from_numpy(np.ascontiguousarray(cloud)).cuda(), cell, device="cuda")
        oc, os_ = O.voxel_downsample(cloud.astype(np.float64), cell)
        G.eq(c, oc, "voxel coords")
        G.eq(s, os_, "voxel sel")
    except Exception as e:
        fails += 1
        print("FAIL seed", seed, repr(e)[:300], flush=True)
print("done", fails, "failures")
