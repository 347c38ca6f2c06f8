"""k_route_count + k_route_scan time (GPU box): 10M int3 keys, world 1..64,
CUDA events, and the per-owner counts checked against a torch bincount of
the owners it wrote."""
import statistics
import sys

sys.path.insert(0, ".")
import torch

from paper_2110_00511_b200 import _lib
from paper_2110_00511_b200.workloads import int3_batch

dev = torch.device("cuda:0")
n = 10_000_000
keys = torch.from_numpy(int3_batch(n, 0.5, seed=7)).to(dev)
st = torch.cuda.current_stream().cuda_stream
for world in (1, 2, 8, 9, 64):
    counts = torch.empty(world, dtype=torch.int64, device=dev)
    owners = torch.empty(n, dtype=torch.uint8, device=dev)
    scratch = torch.empty(int(_lib.lib.ash_route_scratch_len(n, world)), dtype=torch.int32, device=dev)
    ts = []
    for rep in range(12):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        _lib.call("ash_route_count", keys.data_ptr(), n, 3, world, counts.data_ptr(), owners.data_ptr(),
                  scratch.data_ptr(), scratch.numel(), st)
        b.record()
        torch.cuda.synchronize()
        if rep >= 2:
            ts.append(a.elapsed_time(b))
    ok = torch.equal(torch.bincount(owners.long(), minlength=world), counts)
    print(f"world {world:3d}: count+scan median {statistics.median(ts) * 1e3:6.1f} us  counts ok={ok}", flush=True)
