"""Sweep vs direct state stores by table size (GPU box): insert of N int3
keys (rho 0.5) into a fresh capacity-N map, L2 flushed, for the
ASH_SWEEP_TABLE_MIN in the environment (read at load: one process per
setting).  Prints N, table MB and the insert median."""
import os
import statistics
import sys

sys.path.insert(0, ".")
import numpy as np
import torch

import paper_2110_00511_b200 as ash
from paper_2110_00511_b200.workloads import int3_batch

dev = torch.device("cuda:0")
flush = torch.zeros(64 * 1024 * 1024, dtype=torch.float32, device=dev)
for n in (1_000_000, 2_000_000, 3_000_000, 4_000_000, 6_000_000):
    keys = torch.from_numpy(int3_batch(n, 0.5, seed=5)).to(dev)
    vals = torch.rand((n, 1), device=dev)
    m = ash.HashMap(n, 3, [np.float32], device=dev)
    ts = []
    for t in range(12):
        m.clear()
        flush.add_(1)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        m.insert(keys, vals)
        b.record()
        torch.cuda.synchronize()
        if t >= 2:
            ts.append(a.elapsed_time(b))
    print(f"min={os.environ.get('ASH_SWEEP_TABLE_MIN', '-1'):>12s} n={n:>9d} table {m._n_slots * 16 / 2**20:6.1f} MB "
          f"insert {statistics.median(ts):.4f} ms", flush=True)
    del m
