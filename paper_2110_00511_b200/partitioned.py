"""Hash-partitioned map across GPUs (one process per GPU, torch.distributed).

SURVEY §8(e): key ownership is ``owner = mix64(key) mod world`` (independent
of the in-table hash).  Each rank holds a contiguous slice of every global
batch.  A batch op:

  1. stable partition of the local slice by owner (libash route kernels);
  2. exchange counts, then keys (+ value rows) with ``all_to_all_single``
     (NCCL over NVLink on B200; gloo in the CPU tests);
  3. the owner runs the single-GPU op on the received keys — concatenated in
     source-rank order, i.e. in global batch order, so first-occurrence
     winners and masks are bit-exact with one big map;
  4. owner-local indices travel back (``-1`` encodes a False mask, so one
     int32 per key suffices) and are scattered to the original positions.

A global buffer index is the pair ``(owner rank, local index)``; results
carry the owner of every key.  Capacity and auto-rehash are per shard.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch
import torch.distributed as dist

__all__ = ["PartitionedHashMap", "PartitionedResult", "CudaRouter"]


@dataclass
class PartitionedResult:
    indices: torch.Tensor  # owner-local buffer index, -1 where masks is False
    masks: torch.Tensor
    owners: torch.Tensor   # owner rank of every key (uint8)

    def __iter__(self):
        return iter((self.indices, self.masks))

    def __len__(self):
        return len(self.indices)


class CudaRouter:
    """Routing kernels of libash (ash_route.cu) on one device."""

    def __init__(self, world: int, device: torch.device):
        from . import _lib
        self._lib = _lib
        self.world = int(world)
        self.device = device
        self._scratch = torch.empty(0, dtype=torch.int32, device=device)

    def _stream(self):
        return torch.cuda.current_stream(self.device).cuda_stream

    def owners(self, keys: torch.Tensor) -> torch.Tensor:
        out = torch.empty(keys.shape[0], dtype=torch.int32, device=self.device)
        self._lib.call("ash_route_owner", keys.data_ptr(), keys.shape[0], keys.shape[1], self.world,
                       out.data_ptr(), self._stream())
        return out

    def plan(self, keys: torch.Tensor, payloads=()):
        """Partition by owner and build the send buffers in one pass.
        Returns (perm, counts, owners, send_keys, send_payloads)."""
        n = keys.shape[0]
        need = int(self._lib.lib.ash_route_scratch_len(n, self.world))
        if self._scratch.numel() < need:
            self._scratch = torch.empty(max(need, 1), dtype=torch.int32, device=self.device)
        perm = torch.empty(n, dtype=torch.int32, device=self.device)
        counts = torch.empty(self.world, dtype=torch.int64, device=self.device)
        owners = torch.empty(n, dtype=torch.uint8, device=self.device)
        send_keys = torch.empty_like(keys)
        first = payloads[0].contiguous() if payloads else None
        send_first = torch.empty_like(first) if first is not None else None
        rb = first[0].numel() * first.element_size() if (first is not None and n) else 0
        self._lib.call("ash_route_partition", keys.data_ptr(), n, keys.shape[1], self.world,
                       perm.data_ptr(), counts.data_ptr(), owners.data_ptr(), send_keys.data_ptr(),
                       first.data_ptr() if first is not None else None, rb,
                       send_first.data_ptr() if send_first is not None else None,
                       self._scratch.data_ptr(), self._scratch.numel(), self._stream())
        sends = ([send_first] if first is not None else []) + [self.gather(p, perm) for p in payloads[1:]]
        return perm, counts, owners, send_keys, sends

    def gather(self, src: torch.Tensor, perm: torch.Tensor) -> torch.Tensor:
        src = src.contiguous()
        out = torch.empty((perm.shape[0], *src.shape[1:]), dtype=src.dtype, device=self.device)
        rb = src[0].numel() * src.element_size() if src.shape[0] else 0
        self._lib.call("ash_gather_rows", src.data_ptr(), perm.data_ptr(), perm.shape[0], rb,
                       out.data_ptr(), self._stream())
        return out

    def scatter(self, src: torch.Tensor, perm: torch.Tensor) -> torch.Tensor:
        src = src.contiguous()
        out = torch.empty_like(src)
        rb = src[0].numel() * src.element_size() if src.shape[0] else 0
        self._lib.call("ash_scatter_rows", src.data_ptr(), perm.data_ptr(), perm.shape[0], rb,
                       out.data_ptr(), self._stream())
        return out


class PartitionedHashMap:
    """One shard per rank; batch ops are collective (every rank calls them
    with its own slice of the global batch, possibly empty)."""

    def __init__(self, capacity_per_rank: int, key_arity: int, value_specs=(), group=None,
                 device=None, auto_rehash: bool = True, local_map=None, router=None):
        self.group = group
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        self.key_arity = int(key_arity)
        if local_map is None:
            from .hashmap import HashMap
            local_map = HashMap(capacity_per_rank, key_arity, value_specs, auto_rehash=auto_rehash,
                                device=device)
        self.local = local_map
        self.device = getattr(local_map, "device", torch.device("cpu"))
        self.router = router if router is not None else CudaRouter(self.world, self.device)

    # -- routing ---------------------------------------------------------

    def _a2a(self, send: torch.Tensor, send_splits, recv_splits) -> torch.Tensor:
        recv = torch.empty((sum(recv_splits), *send.shape[1:]), dtype=send.dtype, device=send.device)
        dist.all_to_all_single(recv, send, output_split_sizes=recv_splits,
                               input_split_sizes=send_splits, group=self.group)
        return recv

    def _forward(self, keys: torch.Tensor, payloads=()):
        perm, send_counts, owners, skeys, spay = self.router.plan(keys, list(payloads))
        recv_counts = torch.empty_like(send_counts)
        dist.all_to_all_single(recv_counts, send_counts, group=self.group)
        ss, rs = send_counts.tolist(), recv_counts.tolist()
        rkeys = self._a2a(skeys, ss, rs)
        rpay = [self._a2a(p, ss, rs) for p in spay]
        return rkeys, rpay, (perm, ss, rs, owners)

    def _backward(self, local_out: torch.Tensor, ctx) -> torch.Tensor:
        perm, ss, rs, _ = ctx
        back = self._a2a(local_out.contiguous(), rs, ss)
        return self.router.scatter(back, perm)

    def _keys(self, keys) -> torch.Tensor:
        k = torch.as_tensor(np.asarray(keys)) if not isinstance(keys, torch.Tensor) else keys
        if k.dim() == 1 and self.key_arity == 1:
            k = k.reshape(-1, 1)
        if k.dim() != 2 or k.shape[1] != self.key_arity:
            raise ValueError(f"keys must have shape (n, {self.key_arity}), got {tuple(k.shape)}")
        if k.is_floating_point():
            raise ValueError("floating-point keys are not accepted; quantize to int32 first")
        return k.to(device=self.device, dtype=torch.int32).contiguous()

    def _values(self, n, values):
        out = []
        for v in values:
            t = torch.as_tensor(np.asarray(v)) if not isinstance(v, torch.Tensor) else v
            out.append(t.reshape(n, -1).to(self.device).contiguous() if n else
                       t.reshape(0, *t.shape[1:]).to(self.device))
        return out

    def _result(self, idx, ctx) -> PartitionedResult:
        idx = idx.reshape(-1)
        return PartitionedResult(idx, idx >= 0, ctx[3])

    # -- operations --------------------------------------------------------

    def insert(self, keys, *values) -> PartitionedResult:
        keys = self._keys(keys)
        vals = self._values(keys.shape[0], values)
        rkeys, rvals, ctx = self._forward(keys, vals)
        res = self.local.insert(rkeys, *rvals)  # the shard reshapes (n, -1) rows itself
        return self._result(self._backward(torch.as_tensor(res.indices), ctx), ctx)

    def activate(self, keys) -> PartitionedResult:
        keys = self._keys(keys)
        rkeys, _, ctx = self._forward(keys)
        res = self.local.activate(rkeys)
        return self._result(self._backward(torch.as_tensor(res.indices), ctx), ctx)

    def find(self, keys) -> PartitionedResult:
        keys = self._keys(keys)
        rkeys, _, ctx = self._forward(keys)
        res = self.local.find(rkeys)
        return self._result(self._backward(torch.as_tensor(res.indices), ctx), ctx)

    def erase(self, keys) -> torch.Tensor:
        keys = self._keys(keys)
        rkeys, _, ctx = self._forward(keys)
        m = torch.as_tensor(self.local.erase(rkeys)).to(torch.uint8)
        return self._backward(m, ctx).to(torch.bool)

    @property
    def local_size(self) -> int:
        return int(self.local.size)

    @property
    def size(self) -> int:
        t = torch.tensor([self.local_size], dtype=torch.int64, device=self.device)
        dist.all_reduce(t, group=self.group)
        return int(t.item())


# ---------------------------------------------------------------------------
# bench.py entry for N > 1 (torchrun; NCCL)

def bench_main(args, rank: int, world: int) -> None:
    import json
    import os
    import statistics

    from .workloads import int3_batch

    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    dev = torch.device("cuda", local_rank)
    torch.cuda.set_device(dev)
    if "MASTER_ADDR" not in os.environ:  # plain `python bench.py --partitioned`
        import socket
        with socket.socket() as s:
            s.bind(("127.0.0.1", 0))
            os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(s.getsockname()[1]),
                              RANK="0", WORLD_SIZE="1")
    dist.init_process_group("nccl", device_id=dev)
    per_rank = 10_000_000
    rho = 0.5
    # this rank's contiguous slice of the global batch (counter-based keys:
    # distinct across ranks, duplicates within the slice at rate 1 - rho)
    keys = torch.from_numpy(int3_batch(per_rank, rho, seed=1000 + rank)).to(dev)
    vals = torch.rand((per_rank, 1), dtype=torch.float32, device=dev)
    # a shard receives ~per_rank keys per batch (hash-uniform owners): 5%
    # headroom keeps every insert on the no-sync path (batch <= free slots)
    pm = PartitionedHashMap(int(per_rank * 1.05), 3, [np.float32], device=dev)
    flush = torch.zeros(64 * 1024 * 1024, dtype=torch.float32, device=dev)
    stream = torch.cuda.current_stream(dev)

    def step():
        pm.local.clear()
        flush.add_(1)
        dist.barrier()
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record(stream)
        pm.insert(keys, vals)
        pm.find(keys)
        b.record(stream)
        torch.cuda.synchronize()
        return a.elapsed_time(b)

    r = pm.insert(keys, vals)
    f = pm.find(keys)
    assert bool(f.masks.all())
    for _ in range(args.warmup):
        step()
    dist.barrier()
    torch.cuda.synchronize()
    from . import _lib
    launches0 = _lib.lib.ash_launch_count()
    times = [step() for _ in range(args.steps)]
    torch.cuda.synchronize()
    launches = _lib.lib.ash_launch_count() - launches0
    dist.barrier()
    ms = torch.tensor([statistics.mean(times)], dtype=torch.float64, device=dev)
    dist.all_reduce(ms, op=dist.ReduceOp.MAX)
    ms = float(ms.item())
    value = 2 * per_rank * world / (ms / 1e3) / 1e6
    if rank == 0:
        print(json.dumps({
            "metric": "insert & find Mops/s (int3 keys)", "value": round(value, 2), "unit": "Mops/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms, 4),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "int32",
            "data": "synthetic",
            "config": {"workload": f"hash-partitioned map, {per_rank:,} insert + {per_rank:,} find "
                                   f"int3 keys per rank per step (uniqueness {rho}), NCCL all-to-all "
                                   f"routing; step time = max over ranks",
                       "parallelism": f"hash-partitioned x{world}"},
            "gpu_launches": launches,  # libash kernels in the timed region (ash_launch_count)
        }), flush=True)
    dist.destroy_process_group()
