"""k_route_put A/B (GPU box): 10M int3 keys + f32[1] values from one source
into `world` owner buffers (all on this GPU: the store pattern, not NVLink),
staged per-owner runs vs direct row stores (ASH_PUT_STAGED, read at load
time: run once per setting).  Prints the median put time per world size and
checks the rows landed where the direct put puts them.  Then the pull of
one int32 result per position back from the owner buffers (the staged-run
variant of commit 9a67e8a, ASH_PULL_STAGED, is no longer built)."""
import statistics
import sys

sys.path.insert(0, ".")
import numpy as np
import torch

from paper_2110_00511_b200 import _lib
from paper_2110_00511_b200.workloads import int3_batch

dev = torch.device("cuda:0")
n = 10_000_000
keys = torch.from_numpy(int3_batch(n, 0.5, seed=7)).to(dev)
vals = torch.rand((n, 1), device=dev)
st = torch.cuda.current_stream().cuda_stream
for world in (1, 2, 8, 64):
    counts = torch.empty(world, dtype=torch.int64, device=dev)
    owners = torch.empty(n, dtype=torch.uint8, device=dev)
    scratch = torch.empty(int(_lib.lib.ash_route_scratch_len(n, world)), dtype=torch.int32, device=dev)
    _lib.call("ash_route_count", keys.data_ptr(), n, 3, world, counts.data_ptr(), owners.data_ptr(),
              scratch.data_ptr(), scratch.numel(), st)
    C = torch.zeros((world, world), dtype=torch.int64, device=dev)
    C[0] = counts
    cap = int(counts.max()) + 16
    bk = [torch.zeros((cap, 3), dtype=torch.int32, device=dev) for _ in range(world)]
    bp = [torch.zeros((cap, 1), dtype=torch.float32, device=dev) for _ in range(world)]
    P = _lib.c_void_p * world
    pk, pp = P(*[b.data_ptr() for b in bk]), P(*[b.data_ptr() for b in bp])
    jdx = torch.empty(n, dtype=torch.int32, device=dev)
    ts = []
    for rep in range(12):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        _lib.call("ash_route_put_counts", keys.data_ptr(), n, 3, world, 0, owners.data_ptr(), scratch.data_ptr(),
                  scratch.numel(), C.data_ptr(), cap, pk, vals.data_ptr(), 4, pp, jdx.data_ptr(), st)
        b.record()
        torch.cuda.synchronize()
        if rep >= 2:
            ts.append(a.elapsed_time(b))
    # check: owner o's rows are this source's keys of owner o in batch order
    ok = True
    for o in range(world):
        sel = owners == o
        c = int(sel.sum())
        ok &= torch.equal(bk[o][:c], keys[sel]) and torch.equal(bp[o][:c], vals[sel])
    print(f"world {world:3d}: put median {statistics.median(ts) * 1e3:7.1f} us  rows ok={ok}", flush=True)
    res = [torch.arange(cap, dtype=torch.int32, device=dev) * 64 + o for o in range(world)]
    pr = P(*[r.data_ptr() for r in res])
    out = torch.empty(n, dtype=torch.int32, device=dev)
    msk = torch.empty(n, dtype=torch.uint8, device=dev)
    ts = []
    for rep in range(12):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        _lib.call("ash_route_pull_counts", owners.data_ptr(), jdx.data_ptr(), n, world, 0, C.data_ptr(), None,
                  pr, out.data_ptr(), msk.data_ptr(), st)
        b.record()
        torch.cuda.synchronize()
        if rep >= 2:
            ts.append(a.elapsed_time(b))
    own64 = owners.long()
    ok = torch.equal(out, (jdx.long() * 64 + own64).int()) and bool(torch.all(msk == 1))
    print(f"world {world:3d}: pull median {statistics.median(ts) * 1e3:7.1f} us  results ok={ok}", flush=True)
