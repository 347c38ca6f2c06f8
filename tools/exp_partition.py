"""Phase breakdown of the hash-partitioned insert/find at N=1 (GPU box).
NCCL transport: route plan, count exchange (+ host read of the split sizes),
key/value all-to-all, shard op, result all-to-all, un-permute.  Peer
transport (``peer`` argument): dispatch (owner count, count exchange, put
overlapping the host read of the counts, barrier), shard op writing into the
result buffer, combine (barrier, pull, barrier)."""
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
from paper_2110_00511_b200.partitioned import PartitionedHashMap
from paper_2110_00511_b200.workloads import int3_batch

N = 10_000_000
keys = torch.from_numpy(int3_batch(N, 0.5, seed=1000)).to(dev)
vals = torch.rand((N, 1), device=dev)
PEER = "peer" in sys.argv[1:]
pm = PartitionedHashMap(int(N * 1.05), 3, [np.float32], device=dev,
                        transport="peer" if PEER else "nccl")
st = torch.cuda.current_stream()
marks = []


def mark(name):
    e = torch.cuda.Event(enable_timing=True)
    e.record(st)
    marks.append((name, e, time.perf_counter()))


def run():
    marks.clear()
    pm.local.clear()
    torch.cuda.synchronize()
    mark("start")
    k = pm._keys(keys)
    v = pm._values(k.shape[0], [vals])
    perm, sc, owners, sk, sp = pm.router.plan(k, v)
    mark("plan")
    rc = torch.empty_like(sc)
    dist.all_to_all_single(rc, sc)
    ss, rs = sc.tolist(), rc.tolist()
    mark("counts+sync")
    rk = pm._a2a(sk, ss, rs)
    rv = [pm._a2a(p, ss, rs) for p in sp]
    mark("a2a keys+vals")
    res = pm.local.insert(rk, *rv)
    mark("shard insert")
    back = pm._a2a(torch.as_tensor(res.indices).contiguous(), rs, ss)
    mark("a2a back")
    out = pm.router.scatter(back, perm)
    mark("unpermute")
    r = pm.find(keys)
    mark("find (whole)")
    torch.cuda.synchronize()


def run_peer():
    marks.clear()
    pm.local.clear()
    torch.cuda.synchronize()
    mark("start")
    rk, rv, ctx = pm.peer.dispatch(keys, vals)
    mark("dispatch")
    pm.local._op_into("insert", rk, [rv], pm.peer.ret[:rk.shape[0]])
    mark("shard insert")
    pm.peer.combine(None, ctx)
    mark("combine")
    rk, _, ctx = pm.peer.dispatch(keys)
    mark("dispatch")
    pm.local._op_into("find", rk, [], pm.peer.ret[:rk.shape[0]])
    mark("shard find")
    pm.peer.combine(None, ctx)
    mark("combine")
    torch.cuda.synchronize()


for i in range(5):
    (run_peer if PEER else run)()
t = [(n, marks[0][1].elapsed_time(e), 1e3 * (w - marks[0][2])) for n, e, w in marks]
prev = 0
for n, g, h in t[1:]:
    print(f"{n:16s} gpu {g - prev:7.3f} ms (cum {g:7.3f})  host cum {h:7.3f}")
    prev = g
dist.destroy_process_group()
