"""Timeline of one partitioned insert + find at N=1 (GPU box): every kernel
and copy of the step with its start offset, duration and the idle gap
before it (torch.profiler / CUPTI), to see where the routing overhead of
the peer transport goes."""
import sys
import types

sys.path.insert(0, ".")
import torch
import torch.distributed as dist

from paper_2110_00511_b200 import partitioned as P
from paper_2110_00511_b200.workloads import int3_batch

dev = P._bench_init()
args = types.SimpleNamespace(transport=sys.argv[1] if len(sys.argv) > 1 else "peer")
N = 10_000_000
keys = torch.from_numpy(int3_batch(N, 0.5, seed=1000)).to(dev)
vals = torch.rand((N, 1), device=dev)
pm, tr = P._make_pm(args, int(N * 1.05), dev)
flush = torch.zeros(64 * 1024 * 1024, dtype=torch.float32, device=dev)


def step():
    pm.local.clear()
    flush.add_(1)
    torch.cuda.synchronize()
    pm.insert(keys, vals)
    pm.find(keys)
    torch.cuda.synchronize()


for _ in range(5):
    step()
from torch.profiler import ProfilerActivity, profile

with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
    for _ in range(3):
        step()
ev = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
ev.sort(key=lambda e: e.time_range.start)
# split into steps at the flush kernel (the add_)
steps, cur = [], []
for e in ev:
    if "vectorized_elementwise" in e.name and "Add" in e.name or "add" in e.name.lower() and cur and \
            e.time_range.end - e.time_range.start > 20:
        if cur:
            steps.append(cur)
        cur = []
    cur.append(e)
steps.append(cur)
last = steps[-1]
t0 = last[0].time_range.start
prev_end = t0
print(f"transport {tr}; kernels in step: {len(last)}")
for e in last:
    s, d = e.time_range.start - t0, e.time_range.end - e.time_range.start
    gap = e.time_range.start - prev_end
    print(f"{s:9.1f} us  dur {d:8.1f}  gap {gap:7.1f}  {e.name[:90]}")
    prev_end = max(prev_end, e.time_range.end)
print("span", round(prev_end - t0, 1), "us")
dist.destroy_process_group()
