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


@pytest.mark.parametrize("world", [1, 3, 8])
@pytest.mark.parametrize("n", [0, 5000, 200_003])
def test_peer_put_pull_kernels(cuda_ok, world, n):
    """ash_route_put / ash_route_pull with `world` owner buffers on one GPU:
    owner o's buffer holds this rank's owner-o keys and payload rows in batch
    order at row_off[o]; the pull returns owner-buffer values per position."""
    from paper_2110_00511_b200 import _lib
    rng = np.random.default_rng(n + 7 * world)
    k = rng.integers(-2 ** 31, 2 ** 31, size=(n, 3)).astype(np.int32)
    pay = rng.integers(0, 2 ** 31, size=(n, 2)).astype(np.int32)
    own = owner_of_np(k, world)
    dev = torch.device("cuda")
    kt, pt = torch.from_numpy(k).to(dev), torch.from_numpy(pay).to(dev)
    counts = torch.empty(world, dtype=torch.int64, device=dev)
    owners = torch.empty(max(n, 1), dtype=torch.uint8, device=dev)
    scratch = torch.empty(max(int(_lib.lib.ash_route_scratch_len(n, world)), 1), dtype=torch.int32, device=dev)
    st = torch.cuda.current_stream().cuda_stream
    _lib.call("ash_route_count", kt.data_ptr(), n, 3, world, counts.data_ptr(), owners.data_ptr(),
              scratch.data_ptr(), scratch.numel(), st)
    cnt = np.bincount(own, minlength=world)
    assert np.array_equal(counts.cpu().numpy(), cnt)
    row_off = rng.integers(0, 100, size=world)
    bufk = [torch.full((int(row_off[o] + cnt[o]) + 1, 3), -7, dtype=torch.int32, device=dev) for o in range(world)]
    bufp = [torch.zeros((int(row_off[o] + cnt[o]) + 1, 2), dtype=torch.int32, device=dev) for o in range(world)]
    P = _lib.c_void_p * world
    offs = (_lib.ctypes.c_int64 * world)(*row_off.tolist())
    jdx = torch.empty(max(n, 1), dtype=torch.int32, device=dev)
    _lib.call("ash_route_put", kt.data_ptr(), n, 3, world, owners.data_ptr(), scratch.data_ptr(), scratch.numel(),
              offs, P(*[b.data_ptr() for b in bufk]), pt.data_ptr(), 8, P(*[b.data_ptr() for b in bufp]),
              jdx.data_ptr(), st)
    for o in range(world):
        sel = own == o
        got = bufk[o].cpu().numpy()
        assert np.array_equal(got[row_off[o]:row_off[o] + cnt[o]], k[sel])
        assert np.all(got[:row_off[o]] == -7)
        assert np.array_equal(bufp[o].cpu().numpy()[row_off[o]:row_off[o] + cnt[o]], pay[sel])
    ret = [torch.arange(b.shape[0], dtype=torch.int32, device=dev) * 10 + o for o, b in enumerate(bufk)]
    out = torch.empty(max(n, 1), dtype=torch.int32, device=dev)
    msk = torch.empty(max(n, 1), dtype=torch.uint8, device=dev)
    _lib.call("ash_route_pull", owners.data_ptr(), jdx.data_ptr(), n, world, offs,
              P(*[r.data_ptr() for r in ret]), out.data_ptr(), msk.data_ptr(), st)
    if n:
        j = np.zeros(n, np.int64)
        for o in range(world):
            j[own == o] = np.arange(cnt[o])
        expect = (row_off[own] + j) * 10 + own
        assert np.array_equal(out[:n].cpu().numpy(), expect.astype(np.int32))
        assert np.array_equal(msk[:n].cpu().numpy(), (expect >= 0).astype(np.uint8))


def test_partitioned_world1_peer_transport(cuda_ok):
    """The symmetric-memory transport end to end at world size 1 (the put /
    barrier / pull path with this rank as its own peer)."""
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
        rng = np.random.default_rng(4)
        pm = PartitionedHashMap(30_000, 3, [np.float32], device=torch.device("cuda", 0), transport="peer")
        om = OracleMap(30_000, 3, [np.float32])
        for step in range(3):
            keys = rng.integers(-60, 60, size=(40_000, 3)).astype(np.int32)
            vals = rng.random((40_000, 1), dtype=np.float32)
            r, o = pm.insert(keys, vals), om.insert(keys, vals)
            assert np.array_equal(r.indices.cpu().numpy(), o.indices)
            assert np.array_equal(r.masks.cpu().numpy(), o.masks)
            e, oe = pm.erase(keys[::5].copy()), om.erase(keys[::5].copy())
            assert np.array_equal(e.cpu().numpy(), oe)
            a, oa = pm.activate(keys[::-3].copy()), om.activate(keys[::-3].copy())
            assert np.array_equal(a.indices.cpu().numpy(), oa.indices)
            f, of = pm.find(keys[::-1].copy()), om.find(keys[::-1].copy())
            assert np.array_equal(f.indices.cpu().numpy(), of.indices)
        assert pm.size == om.size
        assert pm.local.value_buffer(0).cpu().numpy().tobytes() == om.value_buffer(0).tobytes()
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,rank", [(1, 0), (3, 1), (8, 7)])
def test_peer_put_with_device_count_matrix(cuda_ok, world, rank):
    """ash_route_put_counts: row offsets from the exchanged count matrix on
    the device (rows of earlier sources at each owner); when some owner's
    total passes the receive capacity nothing is stored."""
    from paper_2110_00511_b200 import _lib
    n = 100_003
    rng = np.random.default_rng(world * 10 + rank)
    k = rng.integers(-2 ** 31, 2 ** 31, size=(n, 3)).astype(np.int32)
    pay = rng.integers(0, 2 ** 31, size=(n, 1)).astype(np.int32)
    own = owner_of_np(k, world)
    cnt = np.bincount(own, minlength=world)
    C = rng.integers(0, 5000, size=(world, world)).astype(np.int64)
    C[rank] = cnt
    before = C[:rank].sum(0)
    tot = C.sum(0)
    dev = torch.device("cuda")
    kt, pt = torch.from_numpy(k).to(dev), torch.from_numpy(pay).to(dev)
    counts = torch.empty(world, dtype=torch.int64, device=dev)
    owners = torch.empty(n, dtype=torch.uint8, device=dev)
    scratch = torch.empty(int(_lib.lib.ash_route_scratch_len(n, world)), dtype=torch.int32, device=dev)
    st = torch.cuda.current_stream().cuda_stream
    _lib.call("ash_route_count", kt.data_ptr(), n, 3, world, counts.data_ptr(), owners.data_ptr(),
              scratch.data_ptr(), scratch.numel(), st)
    cap = int(tot.max())
    P = _lib.c_void_p * world
    mat = torch.from_numpy(C).to(dev)
    for capacity, stored in ((cap, True), (cap - 1, False)):
        bufk = [torch.full((cap, 3), -7, dtype=torch.int32, device=dev) for _ in range(world)]
        bufp = [torch.full((cap, 1), -7, dtype=torch.int32, device=dev) for _ in range(world)]
        jdx = torch.empty(n, dtype=torch.int32, device=dev)
        _lib.call("ash_route_put_counts", kt.data_ptr(), n, 3, world, rank, owners.data_ptr(),
                  scratch.data_ptr(), scratch.numel(), mat.data_ptr(), capacity,
                  P(*[b.data_ptr() for b in bufk]), pt.data_ptr(), 4, P(*[b.data_ptr() for b in bufp]),
                  jdx.data_ptr(), st)
        for o in range(world):
            got, gp = bufk[o].cpu().numpy(), bufp[o].cpu().numpy()
            if not stored:
                assert np.all(got == -7) and np.all(gp == -7)
                continue
            sel = own == o
            a, b = int(before[o]), int(before[o] + cnt[o])
            assert np.array_equal(got[a:b], k[sel]) and np.array_equal(gp[a:b], pay[sel])
            assert np.all(got[:a] == -7) and np.all(got[b:] == -7)


@pytest.mark.parametrize("world,rank", [(1, 0), (2, 0), (3, 1), (8, 7), (64, 5)])
@pytest.mark.parametrize("n,shift", [(1, 0), (2047, 0), (2049, 1), (100_003, 0), (100_003, 3)])
def test_peer_pull_with_device_count_matrix(cuda_ok, world, rank, n, shift):
    """ash_route_pull_counts (world > 1: the staged pull, each block's owner
    runs read as 16-byte vectors into shared memory): out[p] = owner o's
    result at (rows of earlier sources at o) + jdx[p], mask = out >= 0; ragged
    tails and unaligned outputs (shift) take the scalar path; an overflowed
    exchange (recv_status[1]) leaves the outputs untouched."""
    from paper_2110_00511_b200 import _lib
    rng = np.random.default_rng(world * 1000 + rank + n + shift)
    k = rng.integers(-2 ** 31, 2 ** 31, size=(n, 3)).astype(np.int32)
    own = owner_of_np(k, world)
    cnt = np.bincount(own, minlength=world)
    C = rng.integers(0, 3000, size=(world, world)).astype(np.int64)
    C[rank] = cnt
    before = C[:rank].sum(0)
    dev = torch.device("cuda")
    kt = torch.from_numpy(k).to(dev)
    counts = torch.empty(world, dtype=torch.int64, device=dev)
    owners = torch.empty(n, dtype=torch.uint8, device=dev)
    scratch = torch.empty(int(_lib.lib.ash_route_scratch_len(n, world)), dtype=torch.int32, device=dev)
    st = torch.cuda.current_stream().cuda_stream
    _lib.call("ash_route_count", kt.data_ptr(), n, 3, world, counts.data_ptr(), owners.data_ptr(),
              scratch.data_ptr(), scratch.numel(), st)
    cap = int(C.sum(0).max())
    P = _lib.c_void_p * world
    mat = torch.from_numpy(C).to(dev)
    bufk = [torch.empty((cap, 3), dtype=torch.int32, device=dev) for _ in range(world)]
    jdx = torch.empty(n, dtype=torch.int32, device=dev)
    _lib.call("ash_route_put_counts", kt.data_ptr(), n, 3, world, rank, owners.data_ptr(),
              scratch.data_ptr(), scratch.numel(), mat.data_ptr(), cap,
              P(*[b.data_ptr() for b in bufk]), 0, 0, P(*([None] * world)), jdx.data_ptr(), st)
    # owner o's results: distinct per (owner, row), some negative (misses)
    res = [torch.from_numpy(np.where(rng.random(cap) < 0.3, -1, np.arange(cap) * 64 + o).astype(np.int32)).to(dev)
           for o in range(world)]
    status = torch.zeros(2, dtype=torch.int32, device=dev)
    out_all = torch.full((n + shift,), -99, dtype=torch.int32, device=dev)
    msk_all = torch.full((n + shift,), 7, dtype=torch.uint8, device=dev)
    out, msk = out_all[shift:], msk_all[shift:]
    for over in (1, 0):
        status[1] = over
        _lib.call("ash_route_pull_counts", owners.data_ptr(), jdx.data_ptr(), n, world, rank, mat.data_ptr(),
                  status.data_ptr(), P(*[r.data_ptr() for r in res]), out.data_ptr(), msk.data_ptr(), st)
        if over:
            assert torch.all(out == -99) and torch.all(msk == 7)
    j = np.zeros(n, np.int64)
    for o in range(world):
        j[own == o] = np.arange(cnt[o])
    resn = [r.cpu().numpy() for r in res]
    expect = np.array([resn[o][before[o] + jj] for o, jj in zip(own, j)], dtype=np.int32)
    assert np.array_equal(out.cpu().numpy(), expect)
    assert np.array_equal(msk.cpu().numpy(), (expect >= 0).astype(np.uint8))
    assert torch.all(out_all[:shift] == -99)


@pytest.mark.parametrize("world", [1, 2, 4, 8])
def test_count_exchange_kernel(cuda_ok, world):
    """ash_route_exchange: every rank's exchange kernel (one per stream, all
    resident together) stores its count row into every peer's buffer and
    waits for theirs; each gets the full matrix and the receive status of
    ash_route_recv_status, over several epochs; an overflow gives status
    [0, 1]."""
    from paper_2110_00511_b200 import _lib
    dev = torch.device("cuda")
    rng = np.random.default_rng(world)
    xchg = [torch.zeros(world * world + world, dtype=torch.int64, device=dev) for _ in range(world)]
    P = _lib.c_void_p * world
    peers = P(*[x.data_ptr() for x in xchg])
    streams = [torch.cuda.Stream() for _ in range(world)]
    torch.cuda.synchronize()
    for epoch in range(1, 4):
        C = rng.integers(0, 1000, size=(world, world)).astype(np.int64)
        cap = int(C.sum(0).max()) - (1 if epoch == 3 else 0)
        counts = [torch.from_numpy(C[r].copy()).to(dev) for r in range(world)]
        mats = [torch.full((world, world), -1, dtype=torch.int64, device=dev) for _ in range(world)]
        stats = [torch.full((2,), -9, dtype=torch.int32, device=dev) for _ in range(world)]
        torch.cuda.synchronize()
        for r in range(world):
            _lib.call("ash_route_exchange", counts[r].data_ptr(), world, r, peers, epoch, cap, mats[r].data_ptr(),
                      stats[r].data_ptr(), 10 ** 10, streams[r].cuda_stream)
        torch.cuda.synchronize()
        for r in range(world):
            assert np.array_equal(mats[r].cpu().numpy(), C), (epoch, r)
            over = epoch == 3
            assert stats[r].tolist() == ([0, 1] if over else [int(C[:, r].sum()), 0])


def test_count_exchange_timeout(cuda_ok):
    """A source that never reaches the exchange: status [0, 2] after the
    timeout instead of a hung kernel."""
    from paper_2110_00511_b200 import _lib
    dev = torch.device("cuda")
    xchg = [torch.zeros(2 * 2 + 2, dtype=torch.int64, device=dev) for _ in range(2)]
    peers = (_lib.c_void_p * 2)(*[x.data_ptr() for x in xchg])
    counts = torch.tensor([3, 4], dtype=torch.int64, device=dev)
    mat = torch.empty((2, 2), dtype=torch.int64, device=dev)
    st = torch.full((2,), -9, dtype=torch.int32, device=dev)
    _lib.call("ash_route_exchange", counts.data_ptr(), 2, 0, peers, 1, 100, mat.data_ptr(), st.data_ptr(),
              5 * 10 ** 6, torch.cuda.current_stream().cuda_stream)
    assert st.tolist() == [0, 2]
    assert xchg[1][2 * 2 + 0].item() == 1 and xchg[1][0:2].tolist() == [3, 4]  # our row + flag reached rank 1
