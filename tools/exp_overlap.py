"""C2 step with the table sweep overlapped with the find (GPU box).

eager:   claim, scan, commit + sweep, find                      (headline)
overlap: claim, scan, commit (deferred); the sweep on a side stream while
         the find runs on the main stream (finds resolve PENDING slots via
         the rank words); the main stream joins the side stream before the
         step's end event, so the sweep is inside the timed region.
Results are checked against the eager step."""
import statistics
import sys

sys.path.insert(0, ".")
import numpy as np
import torch

import paper_2110_00511_b200 as ash
from paper_2110_00511_b200 import _lib
from paper_2110_00511_b200.workloads import gen_keys

N = 10_000_000
dev = torch.device("cuda:0")
keys = torch.from_numpy(gen_keys(N, 0.5, "int3", seed=0)).to(dev)
vals = torch.from_numpy(np.random.default_rng(1).random((N, 1), dtype=np.float32)).to(dev)
m = ash.HashMap(N, 3, [np.float32], device=dev)
flush = torch.zeros(64 * 1024 * 1024, dtype=torch.float32, device=dev)
main = torch.cuda.current_stream(dev)
side = torch.cuda.Stream(dev)
idx = torch.empty(N, dtype=torch.int32, device=dev)
msk = torch.empty(N, dtype=torch.uint8, device=dev)
fidx = torch.empty(N, dtype=torch.int32, device=dev)
fmsk = torch.empty(N, dtype=torch.uint8, device=dev)
vptr = (_lib.c_void_p * 1)(vals.data_ptr())


def step(mode):
    m.clear()
    m._ensure_scan(N)
    flush.add_(1)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(main)
    if mode == "eager":
        _lib.call("ash_insert", m._ptr(), keys.data_ptr(), N, vptr, 0, idx.data_ptr(), msk.data_ptr(), main.cuda_stream)
        _lib.call("ash_find", m._ptr(), keys.data_ptr(), N, fidx.data_ptr(), fmsk.data_ptr(), main.cuda_stream)
    else:
        _lib.call("ash_insert_lazy", m._ptr(), keys.data_ptr(), N, vptr, 0, idx.data_ptr(), msk.data_ptr(),
                  main.cuda_stream)
        ev = torch.cuda.Event()
        ev.record(main)
        side.wait_event(ev)
        _lib.call("ash_settle", m._ptr(), side.cuda_stream)
        _lib.call("ash_find", m._ptr(), keys.data_ptr(), N, fidx.data_ptr(), fmsk.data_ptr(), main.cuda_stream)
        main.wait_stream(side)
    b.record(main)
    torch.cuda.synchronize()
    m._size_known = False
    return a.elapsed_time(b)


ref = None
for mode in ("eager", "overlap", "eager", "overlap"):
    ts = [step(mode) for _ in range(12)][2:]
    out = (idx.clone(), msk.clone(), fidx.clone(), fmsk.clone(), m._slots.clone())
    if ref is None:
        ref = out
    same = all(torch.equal(x, y) for x, y in zip(out, ref))
    print(f"{mode:8s} median {statistics.median(ts):.4f} ms  min {min(ts):.4f}  identical={same}", flush=True)
