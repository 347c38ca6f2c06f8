"""Replays of the golden scenarios recorded from the reference
(oracle/make_golden.py).  Each replay takes a map factory so the same check
runs against the CPU oracle (CPU suite) and the CUDA map (GPU suite)."""
from __future__ import annotations

import hashlib
from pathlib import Path

import numpy as np

from conftest import to_np

GOLDEN = Path(__file__).resolve().parent / "golden"


def load(name):
    return dict(np.load(GOLDEN / f"{name}.npz"))


def eq(a, b, what=""):
    a, b = to_np(a), np.asarray(b)
    assert a.shape == b.shape, f"{what}: shape {a.shape} vs {b.shape}"
    assert np.array_equal(a, b), f"{what}: {np.count_nonzero(a != b)} mismatches"


def bytes_eq(a, b, what=""):
    a, b = np.ascontiguousarray(to_np(a)), np.ascontiguousarray(b)
    assert a.shape == b.shape, f"{what}: shape {a.shape} vs {b.shape}"
    assert a.tobytes() == b.tobytes(), f"{what}: buffer bytes differ"


def replay_trace(make_map):
    g = load("trace_appA")
    a, b, c, d = [1, 1, 1], [2, 2, 2], [3, 3, 3], [4, 4, 4]
    k5, k6, x = [5, 5, 5], [6, 6, 6], [9, 9, 9]
    f32 = np.float32
    m = make_map(8, 3, [np.float32])
    r = m.insert(np.array([a, b, a, c], np.int32), np.array([1, 2, 3, 4], f32))
    eq(r.indices, g["ins1_idx"], "ins1 idx")
    eq(r.masks, g["ins1_mask"], "ins1 mask")
    r = m.activate(np.array([c, d, d, a], np.int32))
    eq(r.indices, g["act_idx"], "act idx")
    eq(r.masks, g["act_mask"], "act mask")
    eq(m.erase(np.array([b, b, x], np.int32)), g["erase_mask"], "erase")
    r = m.insert(np.array([k5, k6], np.int32), np.array([5, 6], f32))
    eq(r.indices, g["ins2_idx"], "ins2 idx")
    m.rehash(16)
    r = m.find(np.array([a, c, d, k5, k6], np.int32))
    eq(r.indices, g["find_idx"], "find idx")
    eq(r.masks, g["find_mask"], "find mask")
    bytes_eq(m.key_buffer, g["key_buffer"], "key buffer")
    bytes_eq(m.value_buffer(0), g["value_buffer"], "value buffer")
    eq(m.active_indices(), g["active"], "active")
    assert m.capacity == int(g["capacity"])


def replay_c1(make_map):
    g = load("c1_insert_find")
    m = make_map(200_000, 3, [np.float32])
    r = m.insert(g["keys"], g["values"])
    eq(r.indices, g["ins_idx"], "insert idx")
    eq(r.masks, g["ins_mask"], "insert mask")
    r = m.find(g["keys"])
    eq(r.indices, g["find_idx"], "find idx")
    eq(r.masks, g["find_mask"], "find mask")
    eq(m.active_indices(), g["active"], "active")
    bytes_eq(m.key_buffer, g["key_buffer"], "key buffer")
    bytes_eq(m.value_buffer(0), g["value_buffer"], "value buffer")
    assert m.size == int(g["size"])


def replay_bindings(make_map):
    g = load("bindings_parity")
    for seed in range(20):
        p = f"s{seed}_"
        keys, vals = g[p + "keys"], g[p + "vals"]
        m = make_map(len(keys), 3, [np.float32])
        r = m.insert(keys, vals)
        eq(r.indices, g[p + "ins_idx"], f"{seed} ins")
        eq(r.masks, g[p + "ins_mask"], f"{seed} ins mask")
        r = m.find(keys)
        eq(r.indices, g[p + "find_idx"], f"{seed} find")
        eq(r.masks, g[p + "find_mask"], f"{seed} find mask")
        eq(m.erase(g[p + "ekeys"]), g[p + "erase"], f"{seed} erase")
        r = m.activate(keys)
        eq(r.indices, g[p + "act_idx"], f"{seed} act")
        eq(r.masks, g[p + "act_mask"], f"{seed} act mask")
        eq(m.active_indices(), g[p + "active"], f"{seed} active")
        bytes_eq(m.key_buffer, g[p + "key_buffer"], f"{seed} key buffer")
        bytes_eq(m.value_buffer(0), g[p + "value_buffer"], f"{seed} value buffer")


def replay_random_ops(make_map, name="random_ops"):
    g = load(name)
    names = sorted(g)
    i = 0

    def take(expect):
        nonlocal i
        key = names[i]
        assert key.split("_", 1)[1] == expect, (key, expect)
        i += 1
        return g[key]

    step = 0
    while i < len(names):
        cap = int(take("capacity0"))
        m = make_map(cap, 3, [((2,), np.float32), np.int32])
        for _ in range(60):
            key = names[i]
            op = key.split("_", 1)[1].rsplit("_keys", 1)[0]
            keys = take(f"{op}_keys")
            if op == "insert":
                v0, v1 = take("v0"), take("v1")
                r = m.insert(keys, v0, v1)
                eq(r.indices, take("idx"), f"step {step} insert idx")
                eq(r.masks, take("mask"), f"step {step} insert mask")
            elif op in ("activate", "find"):
                r = m.activate(keys) if op == "activate" else m.find(keys)
                eq(r.indices, take("idx"), f"step {step} {op} idx")
                eq(r.masks, take("mask"), f"step {step} {op} mask")
            elif op == "erase":
                eq(m.erase(keys), take("mask"), f"step {step} erase")
            else:
                m.rehash(int(take("newcap")))
            assert m.size == int(take("size")), f"step {step} size"
            assert m.capacity == int(take("cap")), f"step {step} capacity"
            step += 1
        eq(m.active_indices(), take("final_active"), "final active")
        bytes_eq(m.key_buffer, take("final_keys"), "final keys")
        bytes_eq(m.value_buffer(0), take("final_v0"), "final v0")
        bytes_eq(m.value_buffer(1), take("final_v1"), "final v1")


def replay_growth(make_map):
    g = load("growth_arity")
    m = make_map(16, 3, [np.float32])
    r = m.insert(g["keys"], g["vals"])
    eq(r.indices, g["ins_idx"], "growth insert idx")
    eq(r.masks, g["ins_mask"], "growth insert mask")
    eq(m.find(g["keys"]).indices, g["find_idx"], "growth find idx")
    assert m.capacity == int(g["capacity"]) == 131072
    for arity in (1, 2, 5, 7):
        k = g[f"a{arity}_keys"]
        mm = make_map(64, arity, [np.int64])
        r = mm.insert(k, np.arange(len(k), dtype=np.int64))
        eq(r.indices, g[f"a{arity}_ins_idx"], f"arity {arity} ins")
        eq(r.masks, g[f"a{arity}_ins_mask"], f"arity {arity} ins mask")
        eq(mm.erase(k[::7]), g[f"a{arity}_erase"], f"arity {arity} erase")
        r = mm.activate(k[::3])
        eq(r.indices, g[f"a{arity}_act_idx"], f"arity {arity} act")
        eq(r.masks, g[f"a{arity}_act_mask"], f"arity {arity} act mask")
        assert mm.capacity == int(g[f"a{arity}_capacity"])
        bytes_eq(mm.value_buffer(0), g[f"a{arity}_value_buffer"], f"arity {arity} values")


def voxel_inputs():
    g = load("voxel")
    pts = np.random.default_rng(707).uniform(-1.2, 1.2, size=(100_000, 3))
    digest = np.frombuffer(hashlib.sha256(pts.tobytes()).digest(), np.uint8)
    assert np.array_equal(digest, g["pts_sha256"]), "regenerated cloud differs"
    return pts, g


def replay_voxel(voxel_fn):
    pts, g = voxel_inputs()
    for s in (0.005, 0.01, 0.05):
        c, sel = voxel_fn(pts, s)
        eq(c, g[f"coords_{s}"], f"coords {s}")
        eq(sel, g[f"sel_{s}"], f"selected {s}")
    c, sel = voxel_fn(g["pts32"], 0.005)
    eq(c, g["coords32"], "coords f32")
    eq(sel, g["sel32"], "selected f32")


def replay_alloc_blocks(make_map, alloc_fn, candidates_fn=None):
    """alloc_fn(global_map, coords) -> (gi, local_map)."""
    g = load("alloc_blocks")
    for shape in ("plane", "sphere"):
        gm = make_map(5000, 3, [((8, 8, 8, 2), np.float32)])
        for f in range(3):
            p = f"{shape}_f{f}_"
            coords = g[p + "coords"]
            if candidates_fn is not None:
                eq(candidates_fn(g[f"{shape}_depth"], g["intr"], g[p + "pose"]), coords,
                   f"{p} candidates")
            gi, local = alloc_fn(gm, coords)
            eq(gi, g[p + "gi"], f"{p} gi")
            eq(local.find(coords).indices, g[p + "local_find_idx"], f"{p} local idx")
            bytes_eq(local.value_buffer(0), g[p + "local_values"], f"{p} local values")
        bytes_eq(gm.key_buffer, g[f"{shape}_global_keys"], f"{shape} global keys")
        eq(gm.active_indices(), g[f"{shape}_global_active"], f"{shape} global active")


def replay_delegate(make_map):
    """make_map(cap, arity, specs, backend) — delegate-backend fixtures:
    App. A capacity case (both backends) and growth + erase + activate."""
    g = load("delegate")
    keys = np.array([[i, i, i] for i in range(8)] + [[0, 0, 0]] * 10, np.int32)
    for b in ("generic", "delegate"):
        m = make_map(8, 3, [np.float32], b)
        r = m.insert(keys, np.arange(len(keys), dtype=np.float32))
        eq(r.indices, g[f"appA_{b}_idx"], f"appA {b} idx")
        eq(r.masks, g[f"appA_{b}_mask"], f"appA {b} mask")
        assert m.capacity == int(g[f"appA_{b}_cap"]), f"appA {b} capacity"
        bytes_eq(m.key_buffer, g[f"appA_{b}_keys"], f"appA {b} key rows")
    k = g["grow_keys"]
    m = make_map(16, 3, [np.int32], "delegate")
    r = m.insert(k, np.arange(len(k), dtype=np.int32))
    eq(r.indices, g["grow_idx"], "grow idx")
    eq(r.masks, g["grow_mask"], "grow mask")
    eq(m.erase(k[::5]), g["grow_erase"], "grow erase")
    r = m.activate(k[::2])
    eq(r.indices, g["grow_act_idx"], "grow activate idx")
    eq(r.masks, g["grow_act_mask"], "grow activate mask")
    assert m.capacity == int(g["grow_cap"])
    bytes_eq(m.key_buffer, g["grow_key_buffer"], "grow key rows (stale loser rows)")
    bytes_eq(m.value_buffer(0), g["grow_values"], "grow values")
    eq(m.active_indices(), g["grow_active"], "grow active")
