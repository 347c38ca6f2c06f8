"""Randomized dedup-select and fused allocation streams against the oracle
(GPU box): voxel_downsample of random clouds (f64 / f32, sizes across the
one-block rank limit), unique_rows, and allocate_blocks sequences into one
global map with random batch sizes (one-block activate vs device insert,
workspace-prefix overflow, growth past capacity), exact.
    python tools/fuzz_dedup.py FIRST_SEED END_SEED"""
import os
import sys

sys.path.insert(0, os.getcwd())
sys.path.insert(0, os.path.join(os.getcwd(), "tests"))
import numpy as np
import torch

import golden_replay as G
import paper_2110_00511_b200 as ash
from oracle import ash_oracle as O
from paper_2110_00511_b200.blocks import unique_rows

fails = 0
for seed in range(int(sys.argv[1]), int(sys.argv[2])):
    rng = np.random.default_rng(seed)
    try:
        # voxelize: n across the small-rank limit (128K positions)
        n = int(rng.choice([1, 31, 33, 1000, 131_071, 131_073, 400_000]))
        dt = np.float64 if rng.random() < 0.7 else np.float32
        pts = (rng.normal(size=(n, 3)) * rng.choice([0.05, 1.0, 30.0])).astype(dt)
        cell = float(rng.choice([0.001, 0.01, 0.2]))
        c, s = ash.voxel_downsample(torch.from_numpy(pts).cuda(), cell, device="cuda")
        oc, os_ = O.voxel_downsample(pts.astype(np.float64), cell)
        G.eq(c, oc, "voxel coords")
        G.eq(s, os_, "voxel sel")
        # unique rows
        m = int(rng.integers(1, 300_000))
        span = int(rng.choice([2, 20, 200, 20_000]))
        rows = rng.integers(-span, span, size=(m, 3)).astype(np.int32)
        u = unique_rows(torch.from_numpy(rows).cuda())
        G.eq(u, rows[O.first_occurrence_mask(rows)], "unique rows")
        # allocate_blocks stream into one global map
        cap = int(rng.integers(16, 50_000))
        gm = ash.HashMap(cap, 3, [((2,), np.float32)], device="cuda")
        og = O.OracleMap(cap, 3, [((2,), np.float32)])
        for step in range(int(rng.integers(2, 8))):
            k = int(rng.integers(1, 200_000))
            sp = int(rng.choice([3, 30, 300]))
            cand = rng.integers(-sp, sp, size=(k, 3)).astype(np.int32)
            gi, _ = ash.allocate_blocks(gm, torch.from_numpy(cand).cuda())
            gi_ref, _, _, _ = O.allocate_blocks_map_calls(og, cand)
            G.eq(gi, gi_ref, f"allocate step {step}")
            assert gm.size == og.size and gm.capacity == og.capacity, (gm.size, og.size, gm.capacity, og.capacity)
        G.bytes_eq(gm.key_buffer, og.key_buffer, "keys")
        gm.validate()
    except Exception as e:
        fails += 1
        print("FAIL seed", seed, repr(e)[:300], flush=True)
print("done", fails, "failures")
