"""Randomized op streams on the hash-partitioned map at world size 1 (GPU
box): both transports (peer memory: device-sized shard ops, the count
exchange kernel, receive-capacity overflow and its redo, shard growth; NCCL
all-to-all), results and shard contents equal to one oracle map.
    python tools/fuzz_part.py FIRST_SEED END_SEED"""
import os
import socket
import sys

sys.path.insert(0, os.getcwd())
import numpy as np
import torch
import torch.distributed as dist

from oracle.ash_oracle import OracleMap
from paper_2110_00511_b200.partitioned import PartitionedHashMap

with socket.socket() as s:
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
dev = torch.device("cuda", 0)
dist.init_process_group("nccl", rank=0, world_size=1, device_id=dev)
fails = 0
for seed in range(int(sys.argv[1]), int(sys.argv[2])):
    rng = np.random.default_rng(seed)
    transport = "peer" if rng.random() < 0.75 else "nccl"
    cap = int(rng.integers(8, 40_000))
    recv = int(rng.integers(4, 60_000))
    try:
        pm = PartitionedHashMap(cap, 3, [np.float32], device=dev, transport=transport, recv_capacity=recv)
        om = OracleMap(cap, 3, [np.float32])
        span = int(rng.choice([5, 40, 400, 4000]))
        for step in range(12):
            op = rng.choice(["insert", "insert", "find", "activate", "erase"])
            n = int(rng.integers(0, 50_000))
            keys = rng.integers(-span, span, size=(n, 3)).astype(np.int32)
            if op == "insert":
                vals = rng.random((n, 1), dtype=np.float32)
                r, o = pm.insert(keys, vals), om.insert(keys, vals)
            elif op == "find":
                r, o = pm.find(keys), om.find(keys)
            elif op == "activate":
                r, o = pm.activate(keys), om.activate(keys)
            else:
                e, oe = pm.erase(keys), om.erase(keys)
                assert np.array_equal(e.cpu().numpy(), oe), "erase"
                continue
            assert np.array_equal(r.indices.cpu().numpy(), o.indices), f"{op} idx"
            assert np.array_equal(r.masks.cpu().numpy(), o.masks), f"{op} mask"
            assert pm.size == om.size, (pm.size, om.size)
        assert pm.local.value_buffer(0)[:om.capacity].cpu().numpy().tobytes() == \
            om.value_buffer(0).tobytes() or pm.local.capacity != om.capacity
        pm.local.validate()
    except Exception as exc:
        fails += 1
        print("FAIL seed", seed, transport, cap, recv, repr(exc)[:300], flush=True)
print("done", fails, "failures")
dist.destroy_process_group()
