"""configs[4] on one GPU (GPU box): the map is built by the mixed stream up
to the last step untimed, then the last step's insert and find kernels are
listed with CUPTI (torch.profiler): where the late, high-load steps spend
their time."""
import sys

sys.path.insert(0, ".")
import numpy as np
import torch
from torch.profiler import ProfilerActivity, profile

import paper_2110_00511_b200 as ash
from paper_2110_00511_b200.workloads import c5_step_counters, keys_from_counters_torch

TOTAL, B = 400_000_000, 1 << 25
dev = torch.device("cuda:0")
m = ash.HashMap(TOTAL, 3, [np.float32], device=dev)
steps = -(-TOTAL // B)


def batch(s):
    ins_c, q_c = c5_step_counters(s * B, min(B, TOTAL - s * B), TOTAL, device=dev)
    return keys_from_counters_torch(ins_c), keys_from_counters_torch(q_c)


for s in list(range(steps - 2)) + [steps - 2]:
    ins, q = batch(s)
    vals = torch.rand((len(ins), 1), device=dev)
    torch.cuda.synchronize()
    if s == steps - 2:
        with profile(activities=[ProfilerActivity.CUDA]) as prof:
            m.insert(ins, vals)
            m.find(q)
            torch.cuda.synchronize()
        ev = sorted([e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA],
                    key=lambda e: e.time_range.start)
        t0 = ev[0].time_range.start
        for e in ev:
            print(f"{e.time_range.start - t0:9.1f} us  dur {e.time_range.end - e.time_range.start:8.1f}  {e.name[:90]}")
        print("load after step:", m.size / (1.5 * TOTAL))
    else:
        m.insert(ins, vals)
        m.find(q)
