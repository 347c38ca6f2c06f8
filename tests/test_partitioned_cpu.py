"""Hash-partitioned mode, world_size 2 over gloo on CPU.

The orchestration (stable partition, count + payload all-to-all, owner-side
op in global batch order, result return and un-permute) is exercised with
CPU stand-ins for the two device pieces: a numpy router (same owner hash as
ash_route.cu, restated here) and the oracle map as the shard.  The claim
under test is SURVEY §8(e): masks and per-key values equal one big map."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle.ash_oracle import OracleMap

M64 = (1 << 64) - 1


def owner_of_np(keys: np.ndarray, world: int) -> np.ndarray:
    """numpy restatement of ash_route.cu owner_of (fmix64 chain)."""
    def fmix(x):
        x ^= x >> np.uint64(33)
        x *= np.uint64(0xff51afd7ed558ccd)
        x ^= x >> np.uint64(33)
        x *= np.uint64(0xc4ceb9fe1a85ec53)
        x ^= x >> np.uint64(33)
        return x
    with np.errstate(over="ignore"):
        x = np.full(len(keys), 0x243F6A8885A308D3 ^ keys.shape[1], dtype=np.uint64)
        for d in range(keys.shape[1]):
            add = np.uint64((0x9E3779B97F4A7C15 * (d + 1)) & M64)
            x = fmix(x ^ (keys[:, d].astype(np.uint32).astype(np.uint64) + add))
        hi = (x >> np.uint64(32)).astype(np.uint64)
        return ((hi * np.uint64(world)) >> np.uint64(32)).astype(np.int32)


class NumpyRouter:
    def __init__(self, world):
        self.world = world

    def owners(self, keys):
        return torch.from_numpy(owner_of_np(keys.numpy(), self.world))

    def plan(self, keys, payloads=()):
        own = owner_of_np(keys.numpy(), self.world)
        perm = torch.from_numpy(np.argsort(own, kind="stable").astype(np.int32))
        counts = np.bincount(own, minlength=self.world).astype(np.int64)
        return (perm, torch.from_numpy(counts), torch.from_numpy(own.astype(np.uint8)),
                self.gather(keys, perm), [self.gather(p, perm) for p in payloads])

    def gather(self, src, perm):
        return src[perm.long()].contiguous()

    def scatter(self, src, perm):
        out = torch.empty_like(src)
        out[perm.long()] = src
        return out


class OracleShard:
    device = torch.device("cpu")

    def __init__(self, cap, arity, specs):
        self.m = OracleMap(cap, arity, specs)

    def _k(self, k):
        return k.numpy()

    def insert(self, keys, *vals):
        return self.m.insert(self._k(keys), *[v.numpy() for v in vals])

    def activate(self, keys):
        return self.m.activate(self._k(keys))

    def find(self, keys):
        return self.m.find(self._k(keys))

    def erase(self, keys):
        return self.m.erase(self._k(keys))

    @property
    def size(self):
        return self.m.size


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, keys_all, vals_all, find_all, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2110_00511_b200.partitioned import PartitionedHashMap
    pm = PartitionedHashMap(len(keys_all), 3, [np.float32], local_map=OracleShard(len(keys_all), 3, [np.float32]),
                            router=NumpyRouter(world))
    sl = np.array_split(np.arange(len(keys_all)), world)[rank]
    fl = np.array_split(np.arange(len(find_all)), world)[rank]
    r = pm.insert(torch.from_numpy(keys_all[sl]), torch.from_numpy(vals_all[sl]))
    f = pm.find(torch.from_numpy(find_all[fl]))
    a = pm.activate(torch.from_numpy(find_all[fl]))
    e = pm.erase(torch.from_numpy(keys_all[sl][::5]))
    # value read back on the owner for this rank's found keys is checked by
    # comparing owner-local indices against the shard's value buffer
    shard_vals = pm.local.m.value_buffer(0)
    found_idx = f.indices.numpy()
    q.put((rank, r.masks.numpy(), f.masks.numpy(), a.masks.numpy(), e.numpy(), f.owners.numpy(),
           found_idx, shard_vals.copy(), pm.local_size, pm.size))
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_partitioned_matches_single_map(world):
    rng = np.random.default_rng(5)
    pool = rng.integers(-50, 50, size=(3000, 3)).astype(np.int32)
    keys = pool[rng.integers(0, len(pool), size=6000)]
    vals = rng.random((len(keys), 1), dtype=np.float32)
    probe = np.concatenate([pool[rng.integers(0, len(pool), size=3000)],
                            rng.integers(60, 90, size=(1000, 3)).astype(np.int32)])
    rng.shuffle(probe)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, keys, vals, probe, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = dict()
    for _ in range(world):
        item = q.get(timeout=300)
        out[item[0]] = item
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    # single-map reference over the whole global batch
    ref = OracleMap(len(keys), 3, [np.float32])
    rins = ref.insert(keys, vals)
    rfind = ref.find(probe)
    ract = ref.activate(probe)
    rer = ref.erase(np.concatenate([keys[s][::5] for s in np.array_split(np.arange(len(keys)), world)]))
    ins = np.concatenate([out[r][1] for r in range(world)])
    fnd = np.concatenate([out[r][2] for r in range(world)])
    act = np.concatenate([out[r][3] for r in range(world)])
    ers = np.concatenate([out[r][4] for r in range(world)])
    assert np.array_equal(ins, rins.masks)
    assert np.array_equal(fnd, rfind.masks)
    assert np.array_equal(act, ract.masks)
    assert np.array_equal(ers, rer)
    # the value stored for every found key equals the single map's
    owners = np.concatenate([out[r][5] for r in range(world)])
    fidx = np.concatenate([out[r][6] for r in range(world)])
    got = np.array([out[o][7][i, 0] if m else np.nan for o, i, m in zip(owners, fidx, fnd)], np.float32)
    want = np.array([ref.value_buffer(0)[i, 0] if m else np.nan for i, m in zip(rfind.indices, rfind.masks)],
                    np.float32)
    assert np.array_equal(got[fnd], want[fnd])
    # shard sizes sum to the single-map size (size is collective)
    assert sum(out[r][8] for r in range(world)) == ref.size
    assert all(out[r][9] == ref.size for r in range(world))


def test_owner_hash_balanced():
    rng = np.random.default_rng(1)
    k = rng.integers(-2 ** 20, 2 ** 20, size=(200_000, 3)).astype(np.int32)
    for world in (2, 4, 8):
        c = np.bincount(owner_of_np(k, world), minlength=world)
        assert c.min() > 0.97 * len(k) / world
