"""Routing kernels (ash_route.cu) vs their numpy restatement, and the
partitioned map end to end on one GPU (world_size 1, NCCL)."""
import os
import socket

import numpy as np
import pytest
import torch

from test_partitioned_cpu import owner_of_np

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def router_cls(cuda_ok):
    from paper_2110_00511_b200.partitioned import CudaRouter
    return CudaRouter


@pytest.mark.parametrize("world", [1, 2, 3, 8, 64])
@pytest.mark.parametrize("n", [0, 1, 1000, 2048, 200_003])
def test_partition_is_stable_owner_sort(router_cls, world, n):
    rng = np.random.default_rng(n + world)
    k = rng.integers(-2 ** 31, 2 ** 31, size=(n, 3)).astype(np.int32)
    r = router_cls(world, torch.device("cuda"))
    kt = torch.from_numpy(k).cuda()
    own = owner_of_np(k, world)
    assert np.array_equal(r.owners(kt).cpu().numpy(), own)
    pay = torch.from_numpy(rng.integers(0, 2 ** 31, size=(n, 5)).astype(np.int32)).cuda()
    pay2 = torch.from_numpy(rng.integers(0, 255, size=(n, 3)).astype(np.uint8)).cuda()
    perm, counts, owners, skeys, spay = r.plan(kt, [pay, pay2])
    order = np.argsort(own, kind="stable")
    assert np.array_equal(perm.cpu().numpy(), order)
    assert np.array_equal(counts.cpu().numpy(), np.bincount(own, minlength=world))
    assert np.array_equal(owners.cpu().numpy(), own.astype(np.uint8))
    assert np.array_equal(skeys.cpu().numpy(), k[order])
    assert np.array_equal(spay[0].cpu().numpy(), pay.cpu().numpy()[order])
    assert np.array_equal(spay[1].cpu().numpy(), pay2.cpu().numpy()[order])
    if n:
        g = r.gather(kt, perm)
        assert np.array_equal(g.cpu().numpy(), k[np.argsort(own, kind="stable")])
        assert np.array_equal(r.scatter(g, perm).cpu().numpy(), k)
        b = torch.from_numpy(rng.integers(0, 255, size=(n, 3)).astype(np.uint8)).cuda()
        assert np.array_equal(r.scatter(r.gather(b, perm), perm).cpu().numpy(), b.cpu().numpy())


def test_partitioned_world1_nccl(cuda_ok):
    import torch.distributed as dist
    from oracle.ash_oracle import OracleMap
    from paper_2110_00511_b200.partitioned import PartitionedHashMap
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        rng = np.random.default_rng(3)
        keys = rng.integers(-100, 100, size=(50_000, 3)).astype(np.int32)
        vals = rng.random((50_000, 1), dtype=np.float32)
        pm = PartitionedHashMap(50_000, 3, [np.float32], device=torch.device("cuda", 0))
        om = OracleMap(50_000, 3, [np.float32])
        r, o = pm.insert(keys, vals), om.insert(keys, vals)
        assert np.array_equal(r.indices.cpu().numpy(), o.indices)
        f, of = pm.find(keys[::-1].copy()), om.find(keys[::-1].copy())
        assert np.array_equal(f.indices.cpu().numpy(), of.indices)
        assert pm.size == om.size
    finally:
        dist.destroy_process_group()
