"""configs[4] through the hash-partitioned map at N=1 (GPU box): GPU time
per phase of each op (dispatch / shard op / combine) with CUDA events, to
compare the peer and NCCL transports at the 2^25-key batch size.
    python tools/exp_c5_peer.py peer|nccl"""
import os, socket, sys, time
sys.path.insert(0, ".")
import numpy as np
import torch
import torch.distributed as dist

with socket.socket() as s:
    s.bind(("127.0.0.1", 0))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(s.getsockname()[1]), RANK="0", WORLD_SIZE="1")
dev = torch.device("cuda:0")
torch.cuda.set_device(dev)
dist.init_process_group("nccl", device_id=dev)
from paper_2110_00511_b200.partitioned import PartitionedHashMap, PeerExchange
from paper_2110_00511_b200.hashmap import HashMap
from paper_2110_00511_b200.workloads import c5_step_batches

transport = sys.argv[1] if len(sys.argv) > 1 else "peer"
total, batch = 400_000_000, 1 << 25
pm = PartitionedHashMap(int(total * 1.05) + (1 << 20), 3, [np.float32], device=dev, transport=transport)
st = torch.cuda.current_stream()
marks = []


def wrap(obj, name, label):
    fn = getattr(obj, name)

    def inner(*a, **k):
        e0 = torch.cuda.Event(enable_timing=True)
        e0.record(st)
        t0 = time.perf_counter()
        r = fn(*a, **k)
        e1 = torch.cuda.Event(enable_timing=True)
        e1.record(st)
        marks.append((label, e0, e1, time.perf_counter() - t0))
        return r
    setattr(obj, name, inner)


if transport == "peer":
    wrap(pm.peer, "dispatch", "dispatch")
    wrap(pm.peer, "combine", "combine")
    wrap(pm.local, "_op_into", "shard op")
else:
    wrap(pm, "_forward", "forward")
    wrap(pm, "_backward", "backward")
    wrap(pm.local, "insert", "shard insert")
    wrap(pm.local, "find", "shard find")
for s in range(-(-total // batch)):
    size = min(batch, total - s * batch)
    ins, q = c5_step_batches(s * batch, size, total, device=dev)
    vals = torch.rand((size, 1), dtype=torch.float32, device=dev)
    torch.cuda.synchronize()
    marks.clear()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(st)
    pm.insert(ins, vals)
    pm.find(q)
    b.record(st)
    torch.cuda.synchronize()
    print(f"step {s}: {a.elapsed_time(b):.3f} ms")
    if s in (6, 10):
        for label, e0, e1, host in marks:
            print(f"   {label:14s} gpu {e0.elapsed_time(e1):7.3f} ms  host {1e3 * host:7.3f} ms")
dist.destroy_process_group()
