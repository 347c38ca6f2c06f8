"""CUPTI timeline of one configs[1] step on the plain map (GPU box): every
kernel of insert + find with its start offset, duration and the idle gap
before it, issued while an L2 flush runs (as in bench.py)."""
import sys

sys.path.insert(0, ".")
import numpy as np
import torch
from torch.profiler import ProfilerActivity, profile

import paper_2110_00511_b200 as ash
from paper_2110_00511_b200.workloads import gen_keys

N = int(sys.argv[1]) if len(sys.argv) > 1 else 10_000_000  # 100000: configs[0]
dev = torch.device("cuda:0")
keys = torch.from_numpy(gen_keys(N, 0.5, "int3", seed=0)).to(dev)
vals = torch.from_numpy(np.random.default_rng(1).random((N, 1), dtype=np.float32)).to(dev)
m = ash.HashMap(N if N >= 1_000_000 else 2 * N, 3, [np.float32], device=dev)  # configs[0]: capacity 2N
flush = torch.zeros(64 * 1024 * 1024, dtype=torch.float32, device=dev)


def step():
    m.clear()
    flush.add_(1)
    m.insert(keys, vals)
    m.find(keys)


for _ in range(5):
    step()
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    step()
    torch.cuda.synchronize()
ev = sorted([e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA],
            key=lambda e: e.time_range.start)
i0 = next(i for i, e in enumerate(ev) if "CUDAFunctorOnSelf_add" in e.name)
t0 = ev[i0].time_range.end
prev = t0
for e in ev[i0 + 1:]:
    print(f"{e.time_range.start - t0:8.1f} us  dur {e.time_range.end - e.time_range.start:7.1f}  "
          f"gap {e.time_range.start - prev:5.1f}  {e.name[:80]}")
    prev = max(prev, e.time_range.end)
print("step after the flush:", round(prev - t0, 1), "us")
