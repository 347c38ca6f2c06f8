"""Peer-memory transport with two ranks sharing one GPU: two processes, a
gloo control plane, receive/result buffers mapped across the processes by
CUDA IPC (torch symmetric memory refuses ranks on one device; the
world-size-1 symmetric test is in test_route_gpu.py), the fused put / pull
routing kernels and the device map as each rank's shard.  Masks and values
equal one big map.  The same two-process runs cover the
NCCL transport's code path (CudaRouter partition kernels, device shard map,
un-permute) with gloo carrying its all_to_all_single (gloo stages CUDA
tensors through the host; NCCL refuses two ranks on one device)."""
import os
import socket

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _transport_kw(transport):
    return dict(transport="peer", peer_mapping="ipc") if transport == "peer" else dict(transport="nccl")


def _worker(rank, world, port, keys_all, vals_all, find_all, q, transport="peer"):
    import sys
    sys.path.insert(0, os.getcwd())
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2110_00511_b200.partitioned import PartitionedHashMap
        dev = torch.device("cuda", 0)
        torch.cuda.set_device(dev)
        pm = PartitionedHashMap(len(keys_all), 3, [np.float32], device=dev, **_transport_kw(transport))
        sl = np.array_split(np.arange(len(keys_all)), world)[rank]
        fl = np.array_split(np.arange(len(find_all)), world)[rank]
        r = pm.insert(keys_all[sl], vals_all[sl])
        f = pm.find(find_all[fl])
        a = pm.activate(find_all[fl])
        e = pm.erase(keys_all[sl][::5].copy())
        torch.cuda.synchronize()
        q.put((rank, r.masks.cpu().numpy(), f.masks.cpu().numpy(), a.masks.cpu().numpy(), e.cpu().numpy(),
               f.owners.cpu().numpy(), f.indices.cpu().numpy(), pm.local.value_buffer(0).cpu().numpy(),
               pm.local_size, None))
    except Exception as exc:  # report instead of hanging the parent
        q.put((rank, "error", repr(exc)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("transport", ["peer", "nccl"])
def test_peer_transport_two_ranks_share_one_gpu(cuda_ok, transport):
    import torch.multiprocessing as mp
    from oracle.ash_oracle import OracleMap
    world = 2
    rng = np.random.default_rng(9)
    pool = rng.integers(-50, 50, size=(3000, 3)).astype(np.int32)
    keys = pool[rng.integers(0, len(pool), size=6000)]
    vals = rng.random((len(keys), 1), dtype=np.float32)
    probe = np.concatenate([pool[rng.integers(0, len(pool), size=3000)],
                            rng.integers(60, 90, size=(1000, 3)).astype(np.int32)])
    rng.shuffle(probe)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, keys, vals, probe, q, transport))
             for r in range(world)]
    for p in procs:
        p.start()
    out = {}
    for _ in range(world):
        item = q.get(timeout=240)
        assert not isinstance(item[1], str), item
        out[item[0]] = item
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    ref = OracleMap(len(keys), 3, [np.float32])
    rins = ref.insert(keys, vals)
    rfind = ref.find(probe)
    ract = ref.activate(probe)
    rer = ref.erase(np.concatenate([keys[s][::5] for s in np.array_split(np.arange(len(keys)), world)]))
    assert np.array_equal(np.concatenate([out[r][1] for r in range(world)]), rins.masks)
    fnd = np.concatenate([out[r][2] for r in range(world)])
    assert np.array_equal(fnd, rfind.masks)
    assert np.array_equal(np.concatenate([out[r][3] for r in range(world)]), ract.masks)
    assert np.array_equal(np.concatenate([out[r][4] for r in range(world)]), rer)
    owners = np.concatenate([out[r][5] for r in range(world)])
    fidx = np.concatenate([out[r][6] for r in range(world)])
    got = np.array([out[o][7][i, 0] if m else np.nan for o, i, m in zip(owners, fidx, fnd)], np.float32)
    want = np.array([ref.value_buffer(0)[i, 0] if m else np.nan for i, m in zip(rfind.indices, rfind.masks)],
                    np.float32)
    assert np.array_equal(got[fnd], want[fnd])
    assert sum(out[r][8] for r in range(world)) == ref.size


def _worker_growth(rank, world, port, batches, vals, q, transport="peer"):
    """Shards that fill (and grow) at different rates: each rank picks its
    own shard op (device-sized or host-checked) while the collectives stay
    identical on every rank."""
    import sys
    sys.path.insert(0, os.getcwd())
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2110_00511_b200.partitioned import PartitionedHashMap
        dev = torch.device("cuda", 0)
        torch.cuda.set_device(dev)
        kw = _transport_kw(transport)
        if transport == "peer":
            kw["recv_capacity"] = 1200
        pm = PartitionedHashMap(1500, 3, [np.float32], device=dev, **kw)
        outs = []
        for b, (keys, v) in enumerate(zip(batches, vals)):
            sl = np.array_split(np.arange(len(keys)), world)[rank]
            r = pm.insert(keys[sl], v[sl])
            f = pm.find(keys[sl][::-1].copy())
            outs.append((r.masks.cpu().numpy(), f.masks.cpu().numpy(), pm.local.capacity))
        torch.cuda.synchronize()
        q.put((rank, outs, pm.local_size))
    except Exception as exc:  # report instead of hanging the parent
        q.put((rank, "error", repr(exc)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("transport", ["peer", "nccl"])
def test_peer_transport_shards_diverge_and_grow(cuda_ok, transport):
    import torch.multiprocessing as mp
    from oracle.ash_oracle import OracleMap
    world = 2
    rng = np.random.default_rng(31)
    batches = [rng.integers(-400, 400, size=(n, 3)).astype(np.int32) for n in (2000, 2300, 4000, 3000)]
    vals = [rng.random((len(b), 1), dtype=np.float32) for b in batches]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker_growth, args=(r, world, port, batches, vals, q, transport))
             for r in range(world)]
    for p in procs:
        p.start()
    out = {}
    for _ in range(world):
        item = q.get(timeout=240)
        assert not isinstance(item[1], str), item
        out[item[0]] = item
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    ref = OracleMap(16, 3, [np.float32])
    for b, (keys, v) in enumerate(zip(batches, vals)):
        ri = ref.insert(keys, v)
        rf = ref.find(keys[np.concatenate([s[::-1] for s in np.array_split(np.arange(len(keys)), world)])])
        got_i = np.concatenate([out[r][1][b][0] for r in range(world)])
        got_f = np.concatenate([out[r][1][b][1] for r in range(world)])
        assert np.array_equal(got_i, ri.masks), b
        assert np.array_equal(got_f, rf.masks), b
    assert sum(out[r][2] for r in range(world)) == ref.size
    caps = [[c for _, _, c in out[r][1]] for r in range(world)]
    assert max(caps[0][-1], caps[1][-1]) > 1500  # the shards grew
