"""Generate golden vectors by running the REFERENCE package itself.

Run in the build container (where /root/reference exists):

    python oracle/make_golden.py

It imports ``spatialhash`` from /root/reference/pkg/src (read-only; nothing
is copied), runs fixed scenarios and writes ``tests/golden/*.npz``.  The
fixtures pin both the CPU oracle (tests/test_oracle_golden.py) and the CUDA
path (tests/test_parity_gpu.py).  /root/reference does not exist on the GPU
box; only the committed .npz files travel.
"""
from __future__ import annotations

import sys
from pathlib import Path

import numpy as np

REF = Path("/root/reference/pkg/src")
OUT = Path(__file__).resolve().parent.parent / "tests" / "golden"


def _ref():
    sys.path.insert(0, str(REF))
    import spatialhash  # noqa: F401
    from spatialhash import HashMap, HashSet, voxel_downsample
    from spatialhash.backends import first_occurrence_unique
    from spatialhash.bench import gen_keys
    from spatialhash.hashing import hash_keys
    from spatialhash.tsdf import TsdfConfig, VoxelBlockGrid
    from spatialhash.tsdf.synthetic import plane_depth, sphere_depth
    from spatialhash.tsdf.types import Frame, Intrinsics
    return dict(HashMap=HashMap, HashSet=HashSet, voxel_downsample=voxel_downsample,
                first_occurrence_unique=first_occurrence_unique, gen_keys=gen_keys,
                hash_keys=hash_keys, TsdfConfig=TsdfConfig, VoxelBlockGrid=VoxelBlockGrid,
                plane_depth=plane_depth, sphere_depth=sphere_depth, Frame=Frame,
                Intrinsics=Intrinsics)


class Recorder:
    """Flat dict of arrays with step-numbered names."""

    def __init__(self):
        self.d = {}
        self.n = 0

    def put(self, name, arr):
        self.d[f"{self.n:04d}_{name}"] = np.asarray(arr)
        self.n += 1


def scenario_trace(R):
    """SURVEY App. A trace, generic backend, plus capacity semantics."""
    HashMap = R["HashMap"]
    a, b, c, d = [1, 1, 1], [2, 2, 2], [3, 3, 3], [4, 4, 4]
    k5, k6, x = [5, 5, 5], [6, 6, 6], [9, 9, 9]
    m = HashMap(8, 3, [np.float32])
    rec = {}
    r = m.insert([a, b, a, c], [1.0, 2.0, 3.0, 4.0])
    rec["ins1_idx"], rec["ins1_mask"] = r.indices, r.masks
    r = m.activate([c, d, d, a])
    rec["act_idx"], rec["act_mask"] = r.indices, r.masks
    rec["erase_mask"] = m.erase([b, b, x])
    r = m.insert([k5, k6], [5.0, 6.0])
    rec["ins2_idx"], rec["ins2_mask"] = r.indices, r.masks
    rec["heap_before_rehash"] = m._heap.heap.copy()
    m.rehash(16)
    r = m.find([a, c, d, k5, k6])
    rec["find_idx"], rec["find_mask"] = r.indices, r.masks
    rec["key_buffer"] = m.key_buffer.copy()
    rec["value_buffer"] = m.value_buffer(0).copy()
    rec["active"] = m.active_indices()
    rec["capacity"] = np.array(m.capacity)
    np.savez_compressed(OUT / "trace_appA.npz", **rec)


def scenario_c1(R):
    """configs[0]: gen_keys(100_000, 0.5, seed=0), f32[1] values from
    default_rng(1), HashMap(200_000, 3, [f32]); insert then find."""
    keys = R["gen_keys"](100_000, 0.5, "int3", seed=0)
    vals = np.random.default_rng(1).random((len(keys), 1), dtype=np.float32)
    m = R["HashMap"](200_000, 3, [np.float32])
    ins = m.insert(keys, vals)
    fnd = m.find(keys)
    np.savez_compressed(
        OUT / "c1_insert_find.npz", keys=keys, values=vals,
        ins_idx=ins.indices, ins_mask=ins.masks, find_idx=fnd.indices,
        find_mask=fnd.masks, active=m.active_indices(),
        key_buffer=m.key_buffer.copy(), value_buffer=m.value_buffer(0).copy(),
        size=np.array(m.size))


def scenario_bindings_parity(R):
    """bindings/tests/test_acceptance_secondary.py:12-49 cases, generic
    backend: full index arrays, masks, active set and buffer bytes."""
    out = {}
    for seed in range(20):
        rng = np.random.default_rng(seed)
        n = int(rng.integers(10, 800))
        pool = rng.integers(-30, 30, size=(max(n // 2, 1), 3)).astype(np.int32)
        keys = pool[rng.integers(0, len(pool), size=n)]
        vals = rng.random((n, 1), dtype=np.float32)
        ekeys = pool[rng.integers(0, len(pool), size=n // 3)]
        m = R["HashMap"](len(keys), 3, value_specs=[np.float32])
        p = f"s{seed}_"
        out[p + "keys"], out[p + "vals"], out[p + "ekeys"] = keys, vals, ekeys
        r = m.insert(keys, vals)
        out[p + "ins_idx"], out[p + "ins_mask"] = r.indices, r.masks
        r = m.find(keys)
        out[p + "find_idx"], out[p + "find_mask"] = r.indices, r.masks
        out[p + "erase"] = m.erase(ekeys)
        r = m.activate(keys)
        out[p + "act_idx"], out[p + "act_mask"] = r.indices, r.masks
        out[p + "active"] = m.active_indices()
        out[p + "key_buffer"] = m.key_buffer.copy()
        out[p + "value_buffer"] = m.value_buffer(0).copy()
    np.savez_compressed(OUT / "bindings_parity.npz", **out)


def scenario_random_ops(R, backend="generic"):
    """Long mixed op sequences (insert / activate / erase / find / rehash)
    over a small key range, recording every output: pins heap recycling
    order (sorted frees), stale rows and auto-rehash growth.  The delegate
    run pins that backend's index rule (heap[top + batch position]), its
    whole-batch transient capacity and the stale key rows of losers."""
    rng = np.random.default_rng(20240817 if backend == "generic" else 5150)
    rec = Recorder()
    for seq in range(6):
        cap = int(rng.integers(4, 40))
        m = R["HashMap"](cap, 3, [((2,), np.float32), np.int32], backend=backend)
        rec.put("capacity0", cap)
        for _ in range(60):
            op = rng.choice(["insert", "insert", "activate", "erase", "find", "rehash"])
            n = int(rng.integers(0, 24))
            keys = rng.integers(-5, 5, size=(n, 3)).astype(np.int32)
            rec.put(f"{op}_keys", keys)
            if op == "insert":
                v0 = rng.random((n, 2), dtype=np.float32)
                v1 = rng.integers(-1000, 1000, size=(n,)).astype(np.int32)
                rec.put("v0", v0)
                rec.put("v1", v1)
                r = m.insert(keys, v0, v1)
                rec.put("idx", r.indices)
                rec.put("mask", r.masks)
            elif op == "activate":
                r = m.activate(keys)
                rec.put("idx", r.indices)
                rec.put("mask", r.masks)
            elif op == "find":
                r = m.find(keys)
                rec.put("idx", r.indices)
                rec.put("mask", r.masks)
            elif op == "erase":
                rec.put("mask", m.erase(keys))
            else:
                newcap = max(2 * m.size, m.size + n, 4)
                rec.put("newcap", newcap)
                m.rehash(newcap)
            rec.put("size", m.size)
            rec.put("cap", m.capacity)
        rec.put("final_active", m.active_indices())
        rec.put("final_keys", m.key_buffer.copy())
        rec.put("final_v0", m.value_buffer(0).copy())
        rec.put("final_v1", m.value_buffer(1).copy())
    name = "random_ops" if backend == "generic" else f"random_ops_{backend}"
    np.savez_compressed(OUT / f"{name}.npz", **rec.d)


def scenario_delegate(R):
    """Delegate backend: the random op streams, App. A's capacity case (8 new
    + 10 duplicate-only keys into capacity 8 grows to 32, generic to 8...16)
    and growth 16 -> 131072 for 1e5 keys."""
    scenario_random_ops(R, "delegate")
    out = {}
    keys = np.array([[i, i, i] for i in range(8)] + [[0, 0, 0]] * 10, np.int32)
    for b in ("generic", "delegate"):
        m = R["HashMap"](8, 3, [np.float32], backend=b)
        r = m.insert(keys, np.arange(len(keys), dtype=np.float32))
        out[f"appA_{b}_idx"], out[f"appA_{b}_mask"] = r.indices, r.masks
        out[f"appA_{b}_cap"] = np.array(m.capacity)
        out[f"appA_{b}_keys"] = m.key_buffer.copy()
    rng = np.random.default_rng(808)
    k = rng.integers(-40, 40, size=(20_000, 3)).astype(np.int32)
    m = R["HashMap"](16, 3, [np.int32], backend="delegate")
    r = m.insert(k, np.arange(len(k), dtype=np.int32))
    e = m.erase(k[::5])
    a = m.activate(k[::2])
    out.update(grow_keys=k, grow_idx=r.indices, grow_mask=r.masks, grow_erase=e, grow_act_idx=a.indices,
               grow_act_mask=a.masks, grow_cap=np.array(m.capacity), grow_key_buffer=m.key_buffer.copy(),
               grow_values=m.value_buffer(0).copy(), grow_active=m.active_indices())
    np.savez_compressed(OUT / "delegate.npz", **out)


def scenario_growth(R):
    """tests/test_acceptance.py:147-161 growth 16 -> 131072, and the
    arity-1 / arity-5 generic paths."""
    rng = np.random.default_rng(606)
    keys = np.unique(rng.integers(-2 ** 24, 2 ** 24, size=(110_000, 3)).astype(np.int32),
                     axis=0)[:100_000]
    rng.shuffle(keys, axis=0)
    vals = np.arange(100_000, dtype=np.float32).reshape(-1, 1)
    m = R["HashMap"](16, 3, [np.float32])
    r = m.insert(keys, vals)
    f = m.find(keys)
    out = dict(keys=keys, vals=vals, ins_idx=r.indices, ins_mask=r.masks,
               find_idx=f.indices, capacity=np.array(m.capacity))
    for arity in (1, 2, 5, 7):
        k = rng.integers(-20, 20, size=(3000, arity)).astype(np.int32)
        mm = R["HashMap"](64, arity, [np.int64])
        v = np.arange(3000, dtype=np.int64)
        r = mm.insert(k, v)
        e = mm.erase(k[::7])
        a = mm.activate(k[::3])
        out[f"a{arity}_keys"] = k
        out[f"a{arity}_ins_idx"], out[f"a{arity}_ins_mask"] = r.indices, r.masks
        out[f"a{arity}_erase"] = e
        out[f"a{arity}_act_idx"], out[f"a{arity}_act_mask"] = a.indices, a.masks
        out[f"a{arity}_capacity"] = np.array(mm.capacity)
        out[f"a{arity}_value_buffer"] = mm.value_buffer(0).copy()
    np.savez_compressed(OUT / "growth_arity.npz", **out)


def scenario_voxel(R):
    """tests/test_acceptance.py:166-172 inputs (seed 707, 1e5 uniform points
    in [-1.2, 1.2]^3 at 5/10/50 mm), plus a float32-widened cloud."""
    rng = np.random.default_rng(707)
    pts = rng.uniform(-1.2, 1.2, size=(100_000, 3))
    # the cloud is regenerated from the seed by the tests; pin its bytes
    import hashlib
    out = {"pts_sha256": np.frombuffer(hashlib.sha256(pts.tobytes()).digest(), np.uint8)}
    for s in (0.005, 0.01, 0.05):
        c, sel = R["voxel_downsample"](pts, s)
        out[f"coords_{s}"], out[f"sel_{s}"] = c, sel
    p32 = np.random.default_rng(5).normal(size=(50_000, 3)).astype(np.float32)
    p32 /= np.linalg.norm(p32, axis=1, keepdims=True)
    c, sel = R["voxel_downsample"](p32.astype(np.float64), 0.005)
    out["pts32"], out["coords32"], out["sel32"] = p32, c, sel
    np.savez_compressed(OUT / "voxel.npz", **out)


def scenario_alloc_blocks(R):
    """tsdf/grid.py:127-150 on 160x120 synthetic plane and sphere frames
    (intrinsics scaled per cli.py:125-130), three frames each with a 2 cm
    x translation per frame; records candidates and every map output."""
    Intr, Frame, Cfg = R["Intrinsics"], R["Frame"], R["TsdfConfig"]
    w, h = 160, 120
    s = w / 320
    intr = Intr(fx=250.0 * s, fy=250.0 * s, cx=(w - 1) / 2, cy=(h - 1) / 2, width=w, height=h)
    cfg = Cfg(0.0058, 8, 0.04)
    out = {}
    for shape in ("plane", "sphere"):
        depth = R["plane_depth"](intr, 1.0) if shape == "plane" else \
            R["sphere_depth"](intr, (0.0, 0.0, 1.0), 0.3)
        grid = R["VoxelBlockGrid"](cfg, capacity=5000)
        out[f"{shape}_depth"] = depth
        for f in range(3):
            pose = np.eye(4)
            pose[0, 3] = 0.02 * f
            fr = Frame(depth.copy(), intr, pose)
            coords = grid._candidate_blocks(fr)
            gi = grid.allocate_blocks(fr)
            p = f"{shape}_f{f}_"
            out[p + "pose"] = pose
            out[p + "coords"] = coords
            out[p + "gi"] = gi
            li, lm = grid.local_map.find(coords)
            out[p + "local_find_idx"] = li
            out[p + "local_values"] = grid.local_map.value_buffer(0).copy()
        out[f"{shape}_global_keys"] = grid.global_map.key_buffer.copy()
        out[f"{shape}_global_active"] = grid.global_map.active_indices()
    out["intr"] = np.array([intr.fx, intr.fy, intr.cx, intr.cy, w, h])
    np.savez_compressed(OUT / "alloc_blocks.npz", **out)


def scenario_hash_dedup(R):
    """hashing.py / backends.py numerics and bench.gen_keys outputs."""
    rng = np.random.default_rng(11)
    out = {}
    for arity in (1, 2, 3, 4, 7):
        k = rng.integers(-2 ** 31, 2 ** 31, size=(500, arity)).astype(np.int32)
        out[f"hash_keys_{arity}"] = k
        for n in (1, 37, 1000, 2 ** 20 + 7):
            out[f"hash_{arity}_{n}"] = R["hash_keys"](k, n)
    for name, (m, lo, hi, ar) in {"fo_small": (300, -3, 3, 3), "fo_big": (20_000, -9, 9, 3),
                                  "fo_a1": (9000, -50, 50, 1), "fo_a5": (6000, -2, 2, 5)}.items():
        k = rng.integers(lo, hi, size=(m, ar)).astype(np.int32)
        out[name + "_keys"] = k
        out[name + "_mask"] = R["first_occurrence_unique"](k)
    for cnt, rho, seed in ((1000, 0.5, 0), (5000, 0.1, 3), (777, 1.0, 9)):
        out[f"gen_{cnt}_{rho}_{seed}"] = R["gen_keys"](cnt, rho, "int3", seed=seed)
    np.savez_compressed(OUT / "hash_dedup.npz", **out)


def scenario_snapshot(R):
    """serialize.py ASHL v1: a snapshot written by the reference after an
    insert / erase / insert sequence (non-trivial heap, two value schemas)."""
    rng = np.random.default_rng(77)
    m = R["HashMap"](64, 3, [((2,), np.float32), ((3,), np.uint8)])
    keys = rng.integers(-9, 9, size=(40, 3)).astype(np.int32)
    v0 = rng.random((40, 2), dtype=np.float32)
    v1 = rng.integers(0, 255, size=(40, 3)).astype(np.uint8)
    m.insert(keys, v0, v1)
    m.erase(keys[::4])
    k2 = rng.integers(-9, 9, size=(10, 3)).astype(np.int32)
    k2v0 = rng.random((10, 2), dtype=np.float32)
    k2v1 = rng.integers(0, 255, size=(10, 3)).astype(np.uint8)
    m.insert(k2, k2v0, k2v1)
    path = OUT / "snapshot_ref.ashl"
    m.save(path, metadata={"note": "golden"})
    np.savez_compressed(OUT / "snapshot.npz", keys=keys, v0=v0, v1=v1, erase=keys[::4], k2=k2,
                        k2v0=k2v0, k2v1=k2v1, snap=np.frombuffer(path.read_bytes(), np.uint8))
    path.unlink()


def main():
    OUT.mkdir(parents=True, exist_ok=True)
    R = _ref()
    only = sys.argv[1:]
    for fn in (scenario_trace, scenario_c1, scenario_bindings_parity, scenario_random_ops,
               scenario_growth, scenario_voxel, scenario_alloc_blocks, scenario_hash_dedup,
               scenario_snapshot, scenario_delegate):
        if only and fn.__name__ not in only:
            continue
        fn(R)
        print("wrote", fn.__name__)


if __name__ == "__main__":
    main()
