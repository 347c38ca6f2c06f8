"""Speculative pending states A/B (GPU box): insert time on configs[1]'s
inputs at rho 0.1 / 0.5 / 1.0 with ASH_SPEC on and off (fresh map per
trial, L2 flushed), results compared between the two."""
import os
import statistics
import sys

sys.path.insert(0, ".")
import numpy as np
import torch

import paper_2110_00511_b200 as ash
from paper_2110_00511_b200.workloads import gen_keys

N = 10_000_000
dev = torch.device("cuda:0")
flush = torch.zeros(64 * 1024 * 1024, dtype=torch.float32, device=dev)
vals = torch.from_numpy(np.random.default_rng(1).random((N, 1), dtype=np.float32)).to(dev)
for rho in (0.1, 0.5, 1.0):
    keys = torch.from_numpy(gen_keys(N, rho, "int3", seed=0)).to(dev)
    m = ash.HashMap(N, 3, [np.float32], device=dev)
    ref = None
    for mode in ("1", "0", "1", "0"):
        os.environ["ASH_SPEC"] = mode
        ts = []
        for trial in range(11):
            m.clear()
            flush.add_(1)
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            r = m.insert(keys, vals)
            b.record()
            torch.cuda.synchronize()
            if trial:
                ts.append(a.elapsed_time(b))
        f = m.find(keys)
        out = (r.indices.clone(), r.masks.clone(), f.indices.clone())
        ref = ref or out
        same = all(torch.equal(x, y) for x, y in zip(out, ref))
        print(f"rho {rho} spec={mode} insert median {statistics.median(ts):.4f} min {min(ts):.4f} same={same}",
              flush=True)
