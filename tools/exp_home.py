"""Table-size experiment: C2 insert + find (10M int3 keys, rho 0.5 / 1.0)
with the table sized at various slots-per-capacity factors (the slot limit
check is disabled, so small factors are valid only while distinct keys fit).
Device-resident keys, L2 flushed, CUDA events."""
import sys
sys.path.insert(0, ".")
import numpy as np
import torch
import paper_2110_00511_b200 as ash
import paper_2110_00511_b200.hashmap as H
from paper_2110_00511_b200.workloads import int3_batch

dev = torch.device("cuda:0")
N = 10_000_000
H._SLOT_LIMIT = 1.0
flush = torch.zeros(64 * 1024 * 1024, dtype=torch.float32, device=dev)
for rho in (0.5, 1.0):
    keys = torch.from_numpy(int3_batch(N, rho, seed=0)).to(dev)
    vals = torch.rand((N, 1), device=dev)
    for f in [float(x) for x in (sys.argv[1:] or ["1.5", "1.0", "0.9", "0.8", "0.7"])]:
        if f * N < rho * N * 1.2:
            continue
        H.TABLE_FACTOR = f
        m = ash.HashMap(N, 3, [np.float32], device=dev)
        ti, tf = [], []
        for i in range(8):
            m.clear()
            flush.add_(1)
            e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
            e[0].record()
            r = m.insert(keys, vals)
            e[1].record()
            fr = m.find(keys)
            e[2].record()
            torch.cuda.synchronize()
            if i >= 3:
                ti.append(e[0].elapsed_time(e[1]))
                tf.append(e[1].elapsed_time(e[2]))
        assert int(r.masks.sum()) == int(np.ceil(rho * N)) and bool(fr.masks.all())
        a, b = np.median(ti), np.median(tf)
        print(f"rho {rho} factor {f}: table {m.slot_count * 16 / 1e6:.0f} MB  insert {a:.3f} ms  "
              f"find {b:.3f} ms  step {a + b:.3f} ms  {2 * N / (a + b) / 1e3:.0f} Mops/s", flush=True)
        del m
