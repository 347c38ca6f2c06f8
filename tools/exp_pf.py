"""Key-row L2 prefetch A/B (GPU box): configs[1] insert and find medians
(fresh map per trial, L2 flushed) for the ASH_PF_CLAIM / ASH_PF_FIND set in
the environment (read when libash loads: one process per setting)."""
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
keys = torch.from_numpy(gen_keys(N, 0.5, "int3", seed=0)).to(dev)
vals = torch.from_numpy(np.random.default_rng(1).random((N, 1), dtype=np.float32)).to(dev)
m = ash.HashMap(N, 3, [np.float32], device=dev)
ti, tf = [], []
for trial in range(13):
    m.clear()
    flush.add_(1)
    a, b, c, d = (torch.cuda.Event(enable_timing=True) for _ in range(4))
    a.record()
    r = m.insert(keys, vals)
    b.record()
    flush.add_(1)
    c.record()
    f = m.find(keys)
    d.record()
    torch.cuda.synchronize()
    if trial >= 3:
        ti.append(a.elapsed_time(b))
        tf.append(c.elapsed_time(d))
assert int(r.masks.sum()) == N // 2 and bool(f.masks.all())
print(f"pf claim {os.environ.get('ASH_PF_CLAIM', '0'):>8s} find {os.environ.get('ASH_PF_FIND', '0'):>8s}: "
      f"insert {statistics.median(ti):.4f} ms  find {statistics.median(tf):.4f} ms", flush=True)
