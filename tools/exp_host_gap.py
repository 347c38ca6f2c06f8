"""Host-induced idle time inside a timed step (GPU box): the same insert +
find timed (a) as bench.py does (GPU idle when the first event fires, so the
host's launch prologue is inside the step) and (b) with a ~2 ms device
sleep queued before the first event (the host has issued the whole step
before the GPU reaches it: device time only).  For the plain map (configs[1]
headline) and the N=1 partitioned map (peer transport)."""
import statistics
import sys

sys.path.insert(0, ".")
import numpy as np
import torch

import paper_2110_00511_b200 as ash
from paper_2110_00511_b200.workloads import int3_batch

N = 10_000_000
dev = torch.device("cuda:0")
stream = torch.cuda.current_stream(dev)
flush = torch.zeros(64 * 1024 * 1024, dtype=torch.float32, device=dev)


def timed(fn, pre_sleep, clear):
    clear()
    flush.add_(1)
    torch.cuda.synchronize()
    if pre_sleep:
        torch.cuda._sleep(4_000_000)  # ~2 ms at 1.9 GHz
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(stream)
    fn()
    b.record(stream)
    torch.cuda.synchronize()
    return a.elapsed_time(b)


def run(name, fn, clear):
    for pre in (False, True, False, True):
        ts = [timed(fn, pre, clear) for _ in range(12)][2:]
        print(f"{name:12s} pre_sleep={pre!s:5s} median {statistics.median(ts):.4f} ms  min {min(ts):.4f}", flush=True)


keys = torch.from_numpy(int3_batch(N, 0.5, seed=1000)).to(dev)
vals = torch.rand((N, 1), device=dev)
m = ash.HashMap(N, 3, [np.float32], device=dev)
run("plain", lambda: (m.insert(keys, vals), m.find(keys)), m.clear)
del m
torch.cuda.empty_cache()
if len(sys.argv) > 1 and sys.argv[1] == "part":
    from paper_2110_00511_b200 import partitioned as P
    import types
    P._bench_init()
    pm, tr = P._make_pm(types.SimpleNamespace(transport="peer"), int(N * 1.05), dev)
    run("partitioned", lambda: (pm.insert(keys, vals), pm.find(keys)), pm.local.clear)
