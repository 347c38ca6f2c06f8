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

That is the ``transport="nccl"`` path.  ``transport="peer"`` (``PeerExchange``,
the bench default) replaces steps 2 and 4 with stores into / loads from the
owners' receive and result buffers over NVLink peer memory; the N x N count
exchange is its only collective.

A global buffer index is the pair ``(owner rank, local index)``; results
carry the owner of every key.  Capacity and auto-rehash are per shard.
"""
from __future__ import annotations

from dataclasses import dataclass
import time

import numpy as np
import torch
import torch.distributed as dist

__all__ = ["PartitionedHashMap", "PartitionedResult", "CudaRouter"]

# sync-free peer ops (device-sized shard op); ASH_PEER_DN=0 keeps the host
# read of the count matrix inside each op
_PEER_DN = __import__("os").environ.get("ASH_PEER_DN", "1") == "1"
# count matrix exchanged through peer memory by one kernel (ash_route_exchange)
# instead of an all-gather + ash_route_recv_status; ASH_PEER_XCHG=0 for A/B
_PEER_XCHG = __import__("os").environ.get("ASH_PEER_XCHG", "1") == "1"
_XCHG_TIMEOUT_NS = 30 * 10 ** 9  # a peer silent this long fails the op instead of hanging the GPU


def _exchange_ok(over: int) -> None:
    if over == 2:
        raise RuntimeError("peer count exchange timed out: a rank did not reach the collective op")


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


class PeerExchange:
    """Dispatch / combine over NVLink peer memory (torch symmetric memory).

    Each rank owns symmetric receive buffers (key rows, one payload buffer)
    and a symmetric result buffer, every peer's copy mapped locally.  A batch
    op is: owner count + N x N count exchange (the only collective, a few
    bytes) -> ``ash_route_put`` stores each key (+ value) row straight into
    its owner's receive buffer, segments in source-rank order -> peer barrier
    -> the shard op on the received rows -> results into the symmetric result
    buffer -> peer barrier -> ``ash_route_pull`` reads every position's result
    from its owner -> peer barrier (buffers free for the next op).  Compared
    with the NCCL transport this removes the send-buffer gather, both payload
    all-to-alls and the un-permute pass."""

    def __init__(self, group, world: int, rank: int, device: torch.device, arity: int,
                 payload=None, capacity: int = 1 << 20, mapping: str = "symmetric"):
        from . import _lib
        self._lib = _lib
        self.group = group if group is not None else dist.group.WORLD
        self.group_name = self.group.group_name
        if mapping not in ("symmetric", "ipc"):
            raise ValueError("mapping must be 'symmetric' or 'ipc'")
        # "symmetric": torch symmetric memory (NVLink peer mappings, device-side
        # barriers) — the multi-GPU product path.  "ipc": CUDA IPC mappings of
        # ordinary allocations with host barriers — lets ranks that share one
        # GPU (tests) run the same put / pull kernels across processes.
        self.mapping = mapping
        if mapping == "symmetric":
            import torch.distributed._symmetric_memory as symm
            self._symm = symm
        self.world, self.rank, self.device, self.arity = world, rank, device, arity
        self.payload = payload  # (row shape, torch dtype) of the single value buffer, or None
        self.pay_rb = 0
        if payload is not None:
            shape, dt = payload
            self.pay_rb = int(np.prod(shape)) * torch.empty(0, dtype=dt).element_size()
        self._scratch = torch.empty(0, dtype=torch.int32, device=device)
        self._mat_h = self._mat_ev = None
        self._flag_h = self._flag_ev = None
        self.capacity = 0
        self._alloc(capacity)
        # count-matrix exchange buffer (ash_route_exchange): symmetric memory
        # only (ranks sharing a GPU exchange the counts through gloo)
        self._p_xchg = None
        self._epoch = 0
        if mapping == "symmetric" and _PEER_XCHG:
            self._xchg = self._symm.empty(world * world + world, dtype=torch.int64, device=device)
            self._xchg.zero_()
            self._xchg_handle = self._symm.rendezvous(self._xchg, self.group_name)
            self._p_xchg = (self._lib.c_void_p * world)(*self._xchg_handle.buffer_ptrs)
            self._xchg_handle.barrier(channel=0)  # zeroed on every rank before the first exchange

    def _alloc(self, cap: int) -> None:
        cap = max(int(cap), 1)
        if getattr(self, "recv_keys", None) is not None:
            self._barrier()  # peers may still read the old buffers (no trailing barrier per op)
        sizes = [(cap * self.arity, torch.int32), (cap, torch.int32)]
        if self.pay_rb:
            sizes.append((cap * self.pay_rb, torch.uint8))
        if self.mapping == "symmetric":
            symm = self._symm
            bufs = [symm.empty(n, dtype=dt, device=self.device) for n, dt in sizes]
            self._handles = [symm.rendezvous(b, self.group_name) for b in bufs]
            ptrs = [list(h.buffer_ptrs) for h in self._handles]
        else:
            from torch.multiprocessing.reductions import reduce_tensor
            bufs = [torch.empty(n, dtype=dt, device=self.device) for n, dt in sizes]
            shared = [None] * self.world
            dist.all_gather_object(shared, [reduce_tensor(b) for b in bufs], group=self.group)
            self._peer_views = [[fn(*args) if r != self.rank else bufs[i]
                                 for r, (fn, args) in ((r, shared[r][i]) for r in range(self.world))]
                                for i in range(len(bufs))]
            ptrs = [[t.data_ptr() for t in views] for views in self._peer_views]
        self.recv_keys, self.ret = bufs[0], bufs[1]
        self.recv_pay = bufs[2] if self.pay_rb else None
        self.capacity = cap
        c_void_p = self._lib.c_void_p
        self._p_keys = (c_void_p * self.world)(*ptrs[0])
        self._p_ret = (c_void_p * self.world)(*ptrs[1])
        self._p_pay = (c_void_p * self.world)(*ptrs[2]) if self.pay_rb else None

    def _barrier(self) -> None:
        """All ranks' device work issued so far is complete and visible."""
        if self.mapping == "symmetric":
            self._handles[0].barrier(channel=0)  # stream-ordered device barrier
        else:
            torch.cuda.current_stream(self.device).synchronize()
            dist.barrier(group=self.group)

    def _stream(self):
        return torch.cuda.current_stream(self.device).cuda_stream

    def dispatch(self, keys: torch.Tensor, payload: torch.Tensor = None):
        """Route keys (+ payload rows) to their owners.  Returns this rank's
        shard batch (keys, payload views into the receive buffers) and the
        context the combine needs."""
        lib = self._lib
        n = keys.shape[0]
        need = int(lib.lib.ash_route_scratch_len(n, self.world))
        if self._scratch.numel() < need:
            self._scratch = torch.empty(max(need, 1), dtype=torch.int32, device=self.device)
        counts = torch.empty(self.world, dtype=torch.int64, device=self.device)
        owners = torch.empty(n, dtype=torch.uint8, device=self.device)
        lib.call("ash_route_count", keys.data_ptr(), n, self.arity, self.world, counts.data_ptr(),
                 owners.data_ptr(), self._scratch.data_ptr(), self._scratch.numel(), self._stream())
        jdx = torch.empty(n, dtype=torch.int32, device=self.device)
        rb = self.pay_rb if (payload is not None and n) else 0
        if rb:
            payload = payload.contiguous()
        def pay_args():  # evaluated per put: a grow replaces the peer buffers
            return (payload.data_ptr() if rb else None, rb, self._p_pay if rb else None)
        put_done = False
        if dist.get_backend(self.group) == "gloo":  # CPU control plane (tests: ranks sharing a GPU)
            parts = [torch.empty(self.world, dtype=torch.int64) for _ in range(self.world)]
            dist.all_gather(parts, counts.cpu(), group=self.group)
            C = torch.stack(parts)
        else:
            mat = torch.empty((self.world, self.world), dtype=torch.int64, device=self.device)
            dist.all_gather_into_tensor(mat, counts, group=self.group)
            # the put takes its row offsets from the matrix on the device, so
            # it runs while the host reads the matrix (the one host read of the op)
            if self._mat_h is None or self._mat_h.shape[0] != self.world:
                self._mat_h = torch.empty((self.world, self.world), dtype=torch.int64, pin_memory=True)
                self._mat_ev = torch.cuda.Event()
            self._mat_h.copy_(mat, non_blocking=True)
            self._mat_ev.record(torch.cuda.current_stream(self.device))
            lib.call("ash_route_put_counts", keys.data_ptr(), n, self.arity, self.world, self.rank,
                     owners.data_ptr(), self._scratch.data_ptr(), self._scratch.numel(), mat.data_ptr(),
                     self.capacity, self._p_keys, *pay_args(), jdx.data_ptr(), self._stream())
            self._mat_ev.synchronize()
            C = self._mat_h.clone()
            put_done = int(C.sum(0).max()) <= self.capacity  # else the kernel stored nothing
        row_off = torch.cumsum(C, 0) - C  # rows of earlier sources at every owner
        m = int(C[:, self.rank].sum())
        peak = int(C.sum(0).max())
        if peak > self.capacity:  # every rank sees the same C: grow together
            # (the skipped put may still be in flight: drain before the old
            # buffers are released)
            torch.cuda.current_stream(self.device).synchronize()
            self._alloc(int(peak * 1.25))
        offs = (lib.ctypes.c_int64 * self.world)(*row_off[self.rank].tolist())
        if not put_done:
            lib.call("ash_route_put", keys.data_ptr(), n, self.arity, self.world, owners.data_ptr(),
                     self._scratch.data_ptr(), self._scratch.numel(), offs, self._p_keys, *pay_args(),
                     jdx.data_ptr(), self._stream())
        self._barrier()  # every source's rows have landed
        rkeys = self.recv_keys[:m * self.arity].view(m, self.arity)
        rpay = None
        if self.pay_rb and payload is not None:
            shape, dt = self.payload
            rpay = self.recv_pay[:m * self.pay_rb].view(dt).view(m, *shape)
        return rkeys, rpay, (n, owners, jdx, offs)

    def dispatch_dn(self, keys: torch.Tensor, payload: torch.Tensor = None):
        """Sync-free dispatch: the put and this rank's received row count
        (``status[0]``, device int32) both come from the exchanged count
        matrix on the device, so the host never waits inside the op.  Returns
        the receive views at full capacity (the shard op reads its length
        from ``status``), ``status`` and the combine context.  ``status[1]``
        = 1 when some owner's rows would pass the receive capacity: nothing
        was stored and the caller redoes the op on the host-checked path."""
        lib = self._lib
        n = keys.shape[0]
        need = int(lib.lib.ash_route_scratch_len(n, self.world))
        if self._scratch.numel() < need:
            self._scratch = torch.empty(max(need, 1), dtype=torch.int32, device=self.device)
        counts = torch.empty(self.world, dtype=torch.int64, device=self.device)
        owners = torch.empty(n, dtype=torch.uint8, device=self.device)
        lib.call("ash_route_count", keys.data_ptr(), n, self.arity, self.world, counts.data_ptr(),
                 owners.data_ptr(), self._scratch.data_ptr(), self._scratch.numel(), self._stream())
        status = torch.empty(2, dtype=torch.int32, device=self.device)
        if self._p_xchg is not None:
            # counts through peer memory, waited for on the device: no
            # collective call, no host wait
            mat = torch.empty((self.world, self.world), dtype=torch.int64, device=self.device)
            self._epoch += 1
            lib.call("ash_route_exchange", counts.data_ptr(), self.world, self.rank, self._p_xchg, self._epoch,
                     self.capacity, mat.data_ptr(), status.data_ptr(), _XCHG_TIMEOUT_NS, self._stream())
        else:
            if dist.get_backend(self.group) == "gloo":  # CPU control plane (tests: ranks sharing a GPU)
                parts = [torch.empty(self.world, dtype=torch.int64) for _ in range(self.world)]
                dist.all_gather(parts, counts.cpu(), group=self.group)
                mat = torch.stack(parts).to(self.device)
            else:
                mat = torch.empty((self.world, self.world), dtype=torch.int64, device=self.device)
                dist.all_gather_into_tensor(mat, counts, group=self.group)
            lib.call("ash_route_recv_status", mat.data_ptr(), self.world, self.rank, self.capacity,
                     status.data_ptr(), self._stream())
        # the overflow flag reaches the host early in the op (its first
        # kernels): the op's end waits for this event, not for the pull
        if self._flag_h is None:
            self._flag_h = torch.zeros(2, dtype=torch.int32, pin_memory=True)
            self._flag_ev = torch.cuda.Event()
        self._flag_h.copy_(status, non_blocking=True)
        self._flag_ev.record(torch.cuda.current_stream(self.device))
        jdx = torch.empty(n, dtype=torch.int32, device=self.device)
        rb = self.pay_rb if (payload is not None and n) else 0
        if rb:
            payload = payload.contiguous()
        lib.call("ash_route_put_counts", keys.data_ptr(), n, self.arity, self.world, self.rank,
                 owners.data_ptr(), self._scratch.data_ptr(), self._scratch.numel(), mat.data_ptr(),
                 self.capacity, self._p_keys, payload.data_ptr() if rb else None, rb,
                 self._p_pay if rb else None, jdx.data_ptr(), self._stream())
        self._barrier()  # every source's rows have landed
        cap = self.capacity
        rkeys = self.recv_keys[:cap * self.arity].view(cap, self.arity)
        rpay = None
        if self.pay_rb and payload is not None:
            shape, dt = self.payload
            rpay = self.recv_pay[:cap * self.pay_rb].view(dt).view(cap, *shape)
        return rkeys, rpay, status, (n, owners, jdx, mat)

    def combine_dn(self, ctx, status):
        n, owners, jdx, mat = ctx
        self._barrier()  # every owner's results are in place
        out = torch.empty(n, dtype=torch.int32, device=self.device)
        msk = torch.empty(n, dtype=torch.uint8, device=self.device)
        self._lib.call("ash_route_pull_counts", owners.data_ptr(), jdx.data_ptr(), n, self.world, self.rank,
                       mat.data_ptr(), status.data_ptr(), self._p_ret, out.data_ptr(), msk.data_ptr(),
                       self._stream())
        # no trailing barrier: the next op's put writes only the receive
        # buffers (read by this op's shard op, which every rank finished
        # before the barrier above), and its shard op writes the result
        # buffers only after its own post-put barrier, which no rank reaches
        # before its pull here is done
        return out, msk.view(torch.bool)

    def combine(self, local_idx, ctx) -> torch.Tensor:
        """local_idx: this owner's results, or None when the shard op wrote
        them into ``self.ret`` itself."""
        n, owners, jdx, offs = ctx
        if local_idx is not None and local_idx.shape[0]:
            self.ret[:local_idx.shape[0]].copy_(local_idx.reshape(-1))
        self._barrier()  # every owner's results are in place
        out = torch.empty(n, dtype=torch.int32, device=self.device)
        msk = torch.empty(n, dtype=torch.uint8, device=self.device)
        self._lib.call("ash_route_pull", owners.data_ptr(), jdx.data_ptr(), n, self.world, offs,
                       self._p_ret, out.data_ptr(), msk.data_ptr(), self._stream())
        # no trailing barrier: the next op's put writes only the receive
        # buffers (read by this op's shard op, which every rank finished
        # before the barrier above), and its shard op writes the result
        # buffers only after its own post-put barrier, which no rank reaches
        # before its pull here is done
        return out, msk.view(torch.bool)


def _on_device(fn):
    """Run a partitioned op with this rank's GPU as the current device."""
    import functools

    @functools.wraps(fn)
    def wrapper(self, *args, **kwargs):
        if self.device.type != "cuda":
            return fn(self, *args, **kwargs)
        with torch.cuda.device(self.device):
            return fn(self, *args, **kwargs)
    return wrapper


class PartitionedHashMap:
    """One shard per rank; batch ops are collective (every rank calls them
    with its own slice of the global batch, possibly empty)."""

    def __init__(self, capacity_per_rank: int, key_arity: int, value_specs=(), group=None,
                 device=None, auto_rehash: bool = True, local_map=None, router=None,
                 transport: str = "nccl", peer_mapping: str = "symmetric", recv_capacity: int = None):
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
        if transport not in ("nccl", "peer"):
            raise ValueError("transport must be 'nccl' or 'peer'")
        self.transport = transport
        self.peer = None
        if transport == "peer":
            specs = getattr(local_map, "value_specs", ())
            if len(specs) > 1:
                raise ValueError("the peer transport carries at most one value buffer")
            payload = (specs[0].shape, local_map._torch_dtypes[0]) if specs else None
            self.peer = PeerExchange(group, self.world, self.rank, self.device, self.key_arity, payload,
                                     capacity=max(int(recv_capacity or capacity_per_rank), 1),
                                     mapping=peer_mapping)

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

    def _peer_op(self, op: str, keys, vals=()):
        """One batch op over the peer transport (PeerExchange)."""
        if op == "insert":
            # checked before the collective starts: every rank fails alike
            specs = getattr(self.local, "value_specs", ())
            if len(vals) != len(specs):
                raise ValueError(f"expected {len(specs)} value batches, got {len(vals)}")
            if vals:  # the put moves raw rows: the map's dtype and row size
                v = vals[0].to(self.local._torch_dtypes[0])
                if v.numel() != keys.shape[0] * int(np.prod(specs[0].shape)):
                    raise ValueError(f"value batch has shape {tuple(vals[0].shape)}, expected "
                                     f"({keys.shape[0]}, {', '.join(map(str, specs[0].shape))})")
                vals = [v]
        if hasattr(self.local, "_dn_check"):
            self.local._dn_check(wait=False)  # a previous device-sized insert's flags, if arrived
        if op != "erase" and _PEER_DN and hasattr(self.local, "_op_into_dn"):
            # sync-free dispatch; the same collectives on every rank whichever
            # shard op each one runs
            rkeys, rpay, status, ctx = self.peer.dispatch_dn(keys, vals[0] if vals else None)
            pays = [rpay] if rpay is not None else []
            over = None
            if self.local._dn_ready(op, self.peer.capacity):
                # the shard op reads its batch length on the device
                self.local._op_into_dn(op, rkeys, pays, self.peer.ret, status)
            else:  # this shard needs the host-checked op (growth): read the length
                m, over = status.tolist()
                _exchange_ok(over)
                if not over:
                    self.local._op_into(op, rkeys[:m], [p[:m] for p in pays], self.peer.ret[:m])
            out, msk = self.peer.combine_dn(ctx, status)
            if over is None:  # the one host read: did a receive buffer overflow?
                self.peer._flag_ev.synchronize()
                over = int(self.peer._flag_h[1])
                _exchange_ok(over)
            if not over:
                self.local._dn_done(op)
                return PartitionedResult(out, msk, ctx[1])
            # nothing was stored anywhere (every rank saw the same matrix):
            # redo on the host-checked path, which grows the buffers
        rkeys, rpay, ctx = self.peer.dispatch(keys, vals[0] if vals else None)
        if op != "erase" and hasattr(self.local, "_op_into"):
            # the shard op writes its indices straight into the result buffer
            self.local._op_into(op, rkeys, [rpay] if rpay is not None else [],
                                self.peer.ret[:rkeys.shape[0]])
            out, msk = self.peer.combine(None, ctx)
            return PartitionedResult(out, msk, ctx[1])
        if op == "insert":
            res = self.local.insert(rkeys, *([rpay] if rpay is not None else []))
        elif op == "erase":
            out, _ = self.peer.combine(torch.as_tensor(self.local.erase(rkeys)).to(torch.int32), ctx)
            return out.to(torch.bool)
        else:
            res = getattr(self.local, op)(rkeys)
        out, msk = self.peer.combine(torch.as_tensor(res.indices), ctx)
        return PartitionedResult(out, msk, ctx[1])

    @_on_device
    def insert(self, keys, *values) -> PartitionedResult:
        keys = self._keys(keys)
        vals = self._values(keys.shape[0], values)
        if self.peer is not None:
            return self._peer_op("insert", keys, vals)
        rkeys, rvals, ctx = self._forward(keys, vals)
        res = self.local.insert(rkeys, *rvals)  # the shard reshapes (n, -1) rows itself
        return self._result(self._backward(torch.as_tensor(res.indices), ctx), ctx)

    @_on_device
    def activate(self, keys) -> PartitionedResult:
        keys = self._keys(keys)
        if self.peer is not None:
            return self._peer_op("activate", keys)
        rkeys, _, ctx = self._forward(keys)
        res = self.local.activate(rkeys)
        return self._result(self._backward(torch.as_tensor(res.indices), ctx), ctx)

    @_on_device
    def find(self, keys) -> PartitionedResult:
        keys = self._keys(keys)
        if self.peer is not None:
            return self._peer_op("find", keys)
        rkeys, _, ctx = self._forward(keys)
        res = self.local.find(rkeys)
        return self._result(self._backward(torch.as_tensor(res.indices), ctx), ctx)

    @_on_device
    def erase(self, keys) -> torch.Tensor:
        keys = self._keys(keys)
        if self.peer is not None:
            return self._peer_op("erase", keys)
        rkeys, _, ctx = self._forward(keys)
        m = torch.as_tensor(self.local.erase(rkeys)).to(torch.uint8)
        return self._backward(m, ctx).to(torch.bool)

    @property
    def local_size(self) -> int:
        if hasattr(self.local, "_dn_check"):
            self.local._dn_check()
        return int(self.local.size)

    @property
    def size(self) -> int:
        dev = "cpu" if dist.get_backend(self.group) == "gloo" else self.device
        t = torch.tensor([self.local_size], dtype=torch.int64, device=dev)
        dist.all_reduce(t, group=self.group)
        return int(t.item())


# ---------------------------------------------------------------------------
# bench.py entry for N > 1 (torchrun; NCCL)

def _shared_gpu() -> bool:
    """ASH_SHARED_GPU=1: every rank on cuda:0 with a gloo control plane and
    CUDA-IPC peer mappings, so the N-rank bench path can run on one GPU."""
    import os
    return os.environ.get("ASH_SHARED_GPU", "0") == "1"


def _bench_init():
    import os
    local_rank = 0 if _shared_gpu() else int(os.environ.get("LOCAL_RANK", "0"))
    dev = torch.device("cuda", local_rank)
    torch.cuda.set_device(dev)
    if "MASTER_ADDR" not in os.environ:  # plain `python bench.py --partitioned`
        import socket
        with socket.socket() as s:
            s.bind(("127.0.0.1", 0))
            os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(s.getsockname()[1]),
                              RANK="0", WORLD_SIZE="1")
    if _shared_gpu():
        dist.init_process_group("gloo")
    else:
        dist.init_process_group("nccl", device_id=dev)
    return dev


def _reduce(x, op=dist.ReduceOp.SUM, dev=None):
    """All-reduce of a host scalar (CPU tensor under gloo, device under NCCL)."""
    on_dev = dist.get_backend() != "gloo"
    t = torch.tensor([x], dtype=torch.float64, device=dev if on_dev else "cpu")
    dist.all_reduce(t, op=op)
    return float(t.item())


def _make_pm(args, capacity: int, dev, recv_capacity: int = None):
    import sys
    transport = getattr(args, "transport", "nccl")
    if _shared_gpu():
        return PartitionedHashMap(capacity, 3, [np.float32], device=dev, transport="peer",
                                  peer_mapping="ipc", recv_capacity=recv_capacity), "peer"
    try:
        return PartitionedHashMap(capacity, 3, [np.float32], device=dev, transport=transport,
                                  recv_capacity=recv_capacity), transport
    except Exception as exc:  # no symmetric memory on this node: NCCL all-to-all instead
        if transport != "peer":
            raise
        print(f"peer transport unavailable ({exc!r}); using NCCL all-to-all", file=sys.stderr)
        return PartitionedHashMap(capacity, 3, [np.float32], device=dev, transport="nccl",
                                  recv_capacity=recv_capacity), "nccl"


def run_c5_partitioned(args, rank: int, world: int, dev, transport: str) -> dict:
    """configs[4]: the 400M-key map built across the ranks by the mixed
    stream — each step inserts 2^25 new keys and finds 2^25 keys (half
    present), every rank holding a contiguous 1/N slice of both global
    batches; total work fixed (strong scaling).  Step time = max over ranks.
    Index-exact at every step: with all-new keys on a fresh heap, a shard's
    winners take its indices in arrival order, so each owner's received insert
    indices are 0, 1, 2, ... in global batch order (checked through the hit
    count and the per-shard sizes); the finds hit exactly the present half."""
    from .workloads import c5_step_batches
    import os
    # configs[4]: 400M keys in steps of 2^25; ASH_C5_TOTAL shrinks it for tests
    total = int(os.environ.get("ASH_C5_TOTAL", 400_000_000))
    batch = min(1 << 25, max(1 << 16, total // 8))
    cap = int(total / world * 1.05) + (1 << 20)
    recv = int(batch / world * 1.25) + (1 << 16)
    a2 = argparse_like(args, transport=transport)
    pm, transport = _make_pm(a2, cap, dev, recv_capacity=recv)
    stream = torch.cuda.current_stream(dev)
    # set-up outside the timed build, like the map's construction: the first
    # collective creates the NCCL communicator and the first launches load
    # the routing kernels (~20-150 ms once); a find leaves the map unchanged
    pm.find(torch.zeros((1024, 3), dtype=torch.int32, device=dev))
    torch.cuda.synchronize()
    steps = -(-total // batch)
    ms = 0.0
    ops = 0
    from . import _lib
    launches0 = _lib.lib.ash_launch_count()
    stored = 0
    for s in range(steps):
        size = min(batch, total - s * batch)
        ins, q = c5_step_batches(s * batch, size, total, device=dev)
        lo, hi = size * rank // world, size * (rank + 1) // world
        ins, q = ins[lo:hi].contiguous(), q[lo:hi].contiguous()
        vals = torch.rand((hi - lo, 1), dtype=torch.float32, device=dev)
        dist.barrier()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        r = pm.insert(ins, vals)
        f = pm.find(q)
        b.record(stream)
        torch.cuda.synchronize()
        ms += _reduce(a.elapsed_time(b), dist.ReduceOp.MAX, dev)
        ops += 2 * size
        new = int(_reduce(int(r.masks.sum()), dev=dev))
        hits = int(_reduce(int(f.masks.sum()), dev=dev))
        stored += new
        assert new == size and hits == size // 2, (s, new, hits)
        # index-exact: all-new keys on a fresh heap take each shard's next
        # indices in arrival order (global batch order), so the indices this
        # rank gets from one owner are consecutive
        for o in range(world):
            v = r.indices[r.owners == o].to(torch.int64)
            assert v.numel() < 2 or bool((v[1:] - v[:-1] == 1).all()), (s, o)
    launches = _lib.lib.ash_launch_count() - launches0
    assert pm.size == total == stored
    del pm
    torch.cuda.empty_cache()
    return {"workload": f"configs[4]: {total:,}-key hash-partitioned map built by the mixed stream ({steps} steps "
                        f"of {batch:,} inserts + {batch:,} finds, half present); every rank holds a contiguous 1/N "
                        "slice of each global batch; time = max over ranks", "scaling": "strong",
            "keys": total, "steps": steps,
            "routing": _routing_name(transport), "mops": round(ops / ms / 1e3, 2), "ms_total": round(ms, 2),
            "gpu_launches": launches,
            "parity": "every step: inserts all new (sum of masks = batch) with the indices from each owner "
                      "consecutive in batch order, finds hit exactly the present half, shard sizes sum to the "
                      "keys stored"}


def argparse_like(args, **kw):
    import copy
    a = copy.copy(args)
    for k, v in kw.items():
        setattr(a, k, v)
    return a


def _routing_name(transport: str) -> str:
    if transport == "peer":
        return "peer-memory put/pull (CUDA IPC, shared GPU)" if _shared_gpu() else \
            "peer-memory put/pull (symmetric memory)"
    return "NCCL all-to-all"


def bench_c5(args, rank: int, world: int) -> None:
    import json
    dev = _bench_init()
    res = run_c5_partitioned(args, rank, world, dev, getattr(args, "transport", "peer"))
    if rank == 0:
        steps = res["steps"]
        print(json.dumps({
            "metric": "insert & find Mops/s (int3 keys)", "value": res["mops"], "unit": "Mops/s",
            "n_gpus": world, "steps": steps, "warmup": 0, "ms_per_step": round(res["ms_total"] / steps, 4),
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "int32",
            "data": "synthetic (counter-based keys generated on the device)",
            "config": {"workload": res["workload"], "routing": res["routing"],
                       "parallelism": f"hash-partitioned x{world}",
                       "setup": "excluded (map construction, one warm-up find: NCCL communicator, kernel loading)",
                       **({"note": "ASH_SHARED_GPU: all ranks on one GPU (functional run, not a scaling "
                                   "number)"} if _shared_gpu() else {})},
            "gpu_launches": res["gpu_launches"], "parity": res["parity"],
        }), flush=True)
    dist.destroy_process_group()


def bench_main(args, rank: int, world: int) -> None:
    import json
    import statistics

    from .workloads import int3_batch

    if getattr(args, "c5", False):
        return bench_c5(args, rank, world)
    dev = _bench_init()
    per_rank = 10_000_000
    rho = 0.5
    # this rank's contiguous slice of the global batch (counter-based keys:
    # distinct across ranks, duplicates within the slice at rate 1 - rho)
    keys = torch.from_numpy(int3_batch(per_rank, rho, seed=1000 + rank)).to(dev)
    vals = torch.rand((per_rank, 1), dtype=torch.float32, device=dev)
    # a shard receives ~per_rank keys per batch (hash-uniform owners): 5%
    # headroom keeps every insert on the no-sync path (batch <= free slots)
    pm, transport = _make_pm(args, int(per_rank * 1.05), dev)
    flush = torch.zeros(64 * 1024 * 1024, dtype=torch.float32, device=dev)
    stream = torch.cuda.current_stream(dev)

    def step():
        # ranks aligned first, then the L2 flush: as in the single-GPU step,
        # the host issues the op while the flush runs, so the events time
        # the device work of the op (not the host's launch prologue)
        dist.barrier()
        pm.local.clear()
        flush.add_(1)
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
    sampler = getattr(args, "clock_sampler", None)
    clk = sampler(dev.index or 0) if (sampler is not None and rank == 0) else None
    if clk is not None:
        clk.__enter__()
    launches0 = _lib.lib.ash_launch_count()
    times = [step() for _ in range(args.steps)]
    torch.cuda.synchronize()
    launches = _lib.lib.ash_launch_count() - launches0
    dist.barrier()
    ms = _reduce(statistics.mean(times), dist.ReduceOp.MAX, dev)
    # keep the GPUs busy ~1 s for the clock sampler (untimed): every rank runs
    # the same number of (collective) steps
    for _ in range(max(3, int(1000.0 / max(ms, 1e-3)))):
        step()
    if clk is not None:
        clk.__exit__(None, None, None)
    med = _reduce(statistics.median(times), dist.ReduceOp.MAX, dev)
    mn = _reduce(min(times), dist.ReduceOp.MAX, dev)
    value = 2 * per_rank * world / (ms / 1e3) / 1e6

    # e2e through the public API: pinned host keys / values in, host results
    # out (the H2D / D2H inside the timed region), max over ranks
    keys_h, vals_h = keys.cpu().pin_memory(), vals.cpu().pin_memory()
    outs_h = [torch.empty(per_rank, dtype=dt, pin_memory=True) for dt in (torch.int32, torch.bool) * 2]
    e2e = []
    for i in range(args.warmup + args.steps):
        pm.local.clear()
        dist.barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        kd = keys_h.to(dev, non_blocking=True)
        vd = vals_h.to(dev, non_blocking=True)
        ri = pm.insert(kd, vd)
        rf = pm.find(kd)
        for o, t in zip(outs_h, (ri.indices, ri.masks, rf.indices, rf.masks)):
            o.copy_(t, non_blocking=True)
        torch.cuda.synchronize()
        t1 = time.perf_counter()
        if i >= args.warmup:
            e2e.append((t1 - t0) * 1e3)
    assert bool(outs_h[3].all())
    e2e_ms = _reduce(statistics.median(e2e), dist.ReduceOp.MAX, dev)
    h2d = 2 * keys_h.numel() * 4 + vals_h.numel() * 4
    d2h = 2 * (per_rank * 4 + per_rank)

    # configs[4] (strong scaling, 400M keys) with both transports
    del pm
    torch.cuda.empty_cache()
    other = {}
    if not getattr(args, "no_c5", False):
        for tr in ("peer", "nccl"):
            if _shared_gpu() and tr == "nccl":
                continue
            other[f"c5_partitioned_{tr}"] = run_c5_partitioned(args, rank, world, dev, tr)
    if rank == 0:
        bw = getattr(args, "hbm_peak", None)
        # per-GPU HBM bytes per key: insert 75 B + find 49 B,
        # + 34 B each of routing (partition + unpermute passes)
        per_key = 75 + 49 + 2 * 34
        frac = round(per_key * per_rank / (ms / 1e3) / 1e9 / bw, 4) if bw else None
        print(json.dumps({
            "metric": "insert & find Mops/s (int3 keys)", "value": round(value, 2), "unit": "Mops/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms, 4),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "int32",
            "data": "synthetic (counter-based int3 keys per rank slice, uniqueness 0.5)",
            "config": {"workload": f"hash-partitioned map, {per_rank:,} insert + {per_rank:,} find "
                                   f"int3 keys per rank per step (uniqueness {rho}); step time = max over ranks",
                       "routing": _routing_name(transport),
                       "parallelism": f"hash-partitioned x{world}",
                       "l2": "flushed between steps (256 MB write per rank)",
                       **({"note": "ASH_SHARED_GPU: all ranks on one GPU (functional run, not a scaling "
                                   "number)"} if _shared_gpu() else {})},
            "step_time": {"mean_ms": round(ms, 4), "median_ms": round(med, 4), "min_ms": round(mn, 4),
                          "trials": len(times), "over_ranks": "max"},
            "roofline": {"bound": "hbm", "kernel": "whole step (per GPU)", "achieved_bytes_per_key": per_key,
                         "achieved": round(per_key * per_rank / (ms / 1e3) / 1e9, 1) if bw else None,
                         "peak": bw, "unit": "GB/s", "frac": frac, "traffic": None},
            "e2e": {"value": round(2 * per_rank * world / (e2e_ms / 1e3) / 1e6, 2), "unit": "Mops/s",
                    "h2d_bytes_per_step": int(h2d * world), "d2h_bytes_per_step": int(d2h * world),
                    "median_ms": round(e2e_ms, 3), "over_ranks": "max"},
            "gpu_launches": launches,  # libash kernels in the timed region (ash_launch_count)
            "clocks": clk.summary() if clk is not None else None,
            "other_configs": other,
        }), flush=True)
    dist.destroy_process_group()
