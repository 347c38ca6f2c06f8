"""Benchmark: insert & find Mops/s on int3 keys (BASELINE.json metric).

Workload at N=1 (BASELINE.json configs[1], the config the metric is quoted
on): a fresh map of capacity 10M, one insert of 10M int3 keys (uniqueness
0.5, one float32 value each), then one find of the same 10M keys.  A step =
that insert + find; value = (insert ops + find ops) / step time.  Map
construction (HashMap.clear) is excluded from the step as in the reference
timing loop (pkg/src/spatialhash/bench.py:110,123).  The working set (keys
120 MB + values 40 MB + table 240 MB) exceeds the 126 MB L2, and L2 is also
flushed between steps.  The line also carries the e2e figure (host in / host
out through the public API), the dominant kernel's roofline, the measured
random-probe ceiling, the CPU baseline, clocks, the libash launch count, the
configs[1] sweep and configs[2..4] in `other_configs`.

Arms:
  default            this repo's CUDA path; one JSON line on rank 0.
  --impl reference   the reference algorithm on the host CPU: the numpy oracle
                     port (oracle/ash_oracle.py; the reference is pure Python
                     and cannot travel to the GPU box) on every host core, the
                     sample sharded by key hash over one process per core.
Multi-GPU (torchrun, N>1): hash-partitioned map, peer-memory routing (NCCL
all-to-all with --transport nccl), 10M insert + 10M find keys per rank per
step (weak scaling).  --c5: configs[4], the 400M-key partitioned map built by
the mixed stream (strong scaling).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

N_KEYS = 10_000_000
RHO = 0.5
CAPACITY = 10_000_000
CPU_SAMPLE_KEYS = int(os.environ.get("ASH_CPU_SAMPLE_KEYS", 1_000_000))  # per host core (sharded by key hash)
METRIC = "insert & find Mops/s (int3 keys)"
UNIT = "Mops/s"


def algorithmic_bytes(op: str, rho_new: float, value_bytes: int, key_bytes: int = 12) -> float:
    """K + 5 + S [+ rho_new (K + 2V + S)], S = 32 B sector."""
    base = key_bytes + 5 + 32
    if op == "find":
        return base
    return base + rho_new * (key_bytes + 2 * value_bytes + 32)


def _profiled_traffic(kernel: str):
    """DRAM bytes per launch of `kernel` from the newest committed ncu summary
    (profiles/<tag>_kernels.json, tools/summarize_profiles.py); None if absent."""
    # newest by capture tag (r01f < r01l < r01r ...): file times do not survive a checkout
    files = sorted((ROOT / "profiles").glob("*_kernels.json"), key=lambda p: p.name)
    for f in reversed(files):
        try:
            d = json.loads(f.read_text())
        except ValueError:
            continue
        if kernel in d and d[kernel].get("dram_bytes_per_launch"):
            return int(d[kernel]["dram_bytes_per_launch"]), f.name
    return None, None


def _random_access(kms):
    files = sorted((ROOT / "profiles").glob("*_random_access.json"))
    if not files:
        return None
    ra = json.loads(files[-1].read_text())
    ceil = ra["probe_32B_gps"]
    find_gps = N_KEYS / (kms["find"] / 1e3) / 1e9
    return {"probe_ceiling_gps": ceil, "source": files[-1].name,
            "find_gprobes_per_s": round(find_gps, 1), "find_frac_of_ceiling": round(find_gps / ceil, 3)}


def _peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return float(d["hbm_gbs"]), "measured"
    return 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks/throttle sampling while the GPU is busy."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "50"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None
        return self

    def __exit__(self, *exc):
        self.lines = []
        if self.proc is not None:
            self.proc.terminate()
            try:
                out, _ = self.proc.communicate(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()
                out, _ = self.proc.communicate()
            self.lines = [l for l in out.splitlines() if l.strip()]
        return False

    def summary(self):
        rows = []
        for l in self.lines:
            f = [x.strip() for x in l.split(",")]
            try:
                rows.append((float(f[0]), float(f[1]), f[4:8]))
            except (ValueError, IndexError):
                continue
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        load = [r for r in rows if r[0] > 0.5 * r[1]] or rows
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        reasons = sorted({n for r in load for n, v in zip(names, r[2]) if v.lower() == "active"})
        return {"sm_mhz": statistics.median(r[0] for r in load), "sm_max_mhz": max(r[1] for r in rows),
                "reasons": reasons, "samples": len(rows), "samples_under_load": len(load)}


# ---------------------------------------------------------------------------
# reference arm: the reference algorithm (numpy oracle port) on host cores

def cpu_reference_step(keys: np.ndarray, vals: np.ndarray):
    from oracle.ash_oracle import OracleMap
    m = OracleMap(len(keys), 3, [np.float32])
    t0 = time.perf_counter()
    m.insert(keys, vals)
    r = m.find(keys)
    dt = time.perf_counter() - t0
    assert bool(r.masks.all())
    return dt


# The reference is single-threaded numpy (its thread pool only splits the
# chain walk, under the GIL).  To give it every host core, the
# CPU arm runs the reference algorithm on P key-hash shards in P processes:
# all copies of a key land in one shard in batch order, so every shard is an
# exact reference map of its keys and the masks equal one big map's.

_SHARD = {}


def _shard_init(keys, vals):
    import os as _os
    for var in ("OMP_NUM_THREADS", "OPENBLAS_NUM_THREADS", "MKL_NUM_THREADS"):
        _os.environ[var] = "1"
    _SHARD["keys"], _SHARD["vals"] = keys, vals


def _shard_step(_):
    return cpu_reference_step(_SHARD["keys"], _SHARD["vals"])


def _owner_shards(keys, vals, parts):
    h = (keys[:, 0].astype(np.uint64) * np.uint64(73856093)) ^ \
        (keys[:, 1].astype(np.uint64) * np.uint64(19349669)) ^ \
        (keys[:, 2].astype(np.uint64) * np.uint64(83492791))
    own = ((h * np.uint64(0x9E3779B97F4A7C15)) >> np.uint64(40)) % np.uint64(parts)
    return [(keys[own == w], vals[own == w]) for w in range(parts)]


class ShardedCpuReference:
    """P worker processes, one reference map per key-hash shard; a step is
    the wall time of all shards' insert + find (started together)."""

    def __init__(self, keys, vals, parts=None):
        import multiprocessing as mp
        import os as _os
        self.parts = parts or len(_os.sched_getaffinity(0))
        self.n = len(keys)
        ctx = mp.get_context("spawn")
        shards = _owner_shards(keys, vals, self.parts)
        self.pools = [ctx.Pool(1, initializer=_shard_init, initargs=sh) for sh in shards]

    def step(self) -> float:
        t0 = time.perf_counter()
        res = [p.apply_async(_shard_step, (0,)) for p in self.pools]
        for r in res:
            r.get()
        return time.perf_counter() - t0

    def close(self):
        for p in self.pools:
            p.terminate()


def run_reference(args, rank: int, world: int):
    if rank != 0:
        return
    cpu = ShardedCpuReference(*_cpu_sample())
    try:
        for _ in range(args.warmup):
            cpu.step()
        times = [cpu.step() for _ in range(args.steps)]
    finally:
        cpu.close()
    t = sum(times) / len(times)
    value = 2 * cpu.n / t / 1e6
    sample = (f"per step: insert+find of {cpu.n:,} int3 keys (rho={RHO}, f32[1]) split by key hash "
              f"over {cpu.parts} processes, each a fresh reference map of its shard (the reference "
              f"generic-backend algorithm, numpy oracle port, one core per process)")
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": round(value, 4), "unit": UNIT,
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(t * 1e3, 3), "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "int32", "data": "synthetic",
        "config": {"workload": f"C2 sample: {cpu.n:,} int3 keys rho={RHO} f32[1] insert+find, "
                               f"{cpu.parts} key-hash shards", "capacity": cpu.n},
        "cpu_baseline": {"value": round(value, 4), "unit": UNIT, "cores": cpu.parts, "kind": "port",
                         "sample": sample},
        "e2e": {"value": round(value, 4), "unit": UNIT, "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }), flush=True)


# ---------------------------------------------------------------------------
# GPU arm

class Events:
    def __init__(self, torch, stream):
        self.torch = torch
        self.stream = stream
        self.pairs = []

    def start(self):
        e = self.torch.cuda.Event(enable_timing=True)
        e.record(self.stream)
        return e

    def stop(self, s):
        e = self.torch.cuda.Event(enable_timing=True)
        e.record(self.stream)
        self.pairs.append((s, e))

    def total_ms(self):
        self.torch.cuda.synchronize()
        return sum(s.elapsed_time(e) for s, e in self.pairs)


def l2_flush(torch, buf):
    buf.add_(1)  # 256 MB read+write > 126 MB L2


def gpu_single(args, torch, dev):
    """N=1: the plain map (no routing)."""
    import paper_2110_00511_b200 as ash
    from paper_2110_00511_b200 import _lib
    from paper_2110_00511_b200.workloads import int3_batch

    stream = torch.cuda.current_stream(dev)
    keys_np = int3_batch(N_KEYS, RHO, seed=0)
    vals_np = np.random.default_rng(1).random((N_KEYS, 1), dtype=np.float32)
    keys_h = torch.from_numpy(keys_np).pin_memory()
    vals_h = torch.from_numpy(vals_np).pin_memory()
    keys = keys_h.to(dev)
    vals = vals_h.to(dev)
    flush = torch.zeros(64 * 1024 * 1024, dtype=torch.float32, device=dev)
    m = ash.HashMap(CAPACITY, 3, [np.float32], device=dev)

    def step(ev):
        m.clear()
        l2_flush(torch, flush)
        s = ev.start()
        m.insert(keys, vals)
        m.find(keys)
        ev.stop(s)

    # correctness backstop (reference bench.py:134-150)
    m.clear()
    r = m.insert(keys, vals)
    f = m.find(keys)
    n_unique = int(np.ceil(RHO * N_KEYS))
    assert m.size == n_unique and int(r.masks.sum()) == n_unique and bool(f.masks.all())

    warm = Events(torch, stream)
    for _ in range(args.warmup):
        step(warm)
    torch.cuda.synchronize()
    timed = Events(torch, stream)
    with ClockSampler(dev.index or 0) as clk:
        torch.cuda.synchronize()
        launches0 = _lib.lib.ash_launch_count()
        for _ in range(args.steps):
            step(timed)
        torch.cuda.synchronize()
        launches = _lib.lib.ash_launch_count() - launches0
        # keep the GPU busy for the clock sampler: extra untimed steps
        extra = Events(torch, stream)
        t_end = time.time() + (0.0 if args.profile else 1.0)
        while time.time() < t_end:
            step(extra)
        torch.cuda.synchronize()
    ms = timed.total_ms() / args.steps
    value = 2 * N_KEYS / (ms / 1e3) / 1e6
    if args.profile:
        print(json.dumps({"profile_ms_per_step": ms, "value": value}), flush=True)
        sys.exit(0)

    # per-kernel split (same workload): claim / commit / find, CUDA events on
    # the launching stream
    kern = {"claim": [], "tile_scan": [], "commit": [], "find": []}
    for _ in range(5):
        m.clear()
        l2_flush(torch, flush)
        idx = torch.empty(N_KEYS, dtype=torch.int32, device=dev)
        msk = torch.empty(N_KEYS, dtype=torch.uint8, device=dev)
        vptr = (_lib.c_void_p * 1)(vals.data_ptr())
        m._ensure_scan(N_KEYS)
        e = [torch.cuda.Event(enable_timing=True) for _ in range(5)]
        e[0].record(stream)
        _lib.call("ash_insert_claim", m._ptr(), keys.data_ptr(), N_KEYS, idx.data_ptr(), msk.data_ptr(), m._stream())
        e[1].record(stream)
        _lib.call("ash_insert_count", m._ptr(), N_KEYS, idx.data_ptr(), msk.data_ptr(), m._stream())
        e[2].record(stream)
        _lib.call("ash_insert_commit", m._ptr(), keys.data_ptr(), N_KEYS, vptr, 0, idx.data_ptr(), msk.data_ptr(), m._stream())
        e[3].record(stream)
        m._size_known = False
        l2_flush(torch, flush)
        e4 = torch.cuda.Event(enable_timing=True)
        e4.record(stream)
        m.find(keys)
        e[4].record(stream)
        torch.cuda.synchronize()
        kern["claim"].append(e[0].elapsed_time(e[1]))
        kern["tile_scan"].append(e[1].elapsed_time(e[2]))
        kern["commit"].append(e[2].elapsed_time(e[3]))
        kern["find"].append(e4.elapsed_time(e[4]))
    kms = {k: statistics.median(v) for k, v in kern.items()}

    # e2e: public API with pinned host buffers; H2D of inputs and D2H of the
    # results inside the timed region
    # The API returns host results for host keys (the D2H is inside the call
    # and the call returns only when the results are on the host), so the
    # step is timed on the host clock around the two calls.
    e2e = []
    for i in range(args.warmup + args.steps):
        m.clear()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        r = m.insert(keys_h, vals_h)
        f = m.find(keys_h)
        t1 = time.perf_counter()
        assert not r.indices.is_cuda and not f.masks.is_cuda
        if i >= args.warmup:
            e2e.append((t1 - t0) * 1e3)
    assert int(r.masks.sum()) == int(np.ceil(RHO * N_KEYS)) and bool(f.masks.all())
    e2e_ms = sum(e2e) / len(e2e)
    h2d = 2 * keys_np.nbytes + vals_np.nbytes
    d2h = 2 * (r.indices.numel() * 4 + r.masks.numel())

    sweep = run_sweep(torch, dev, ash, flush)
    other = run_other_configs(torch, dev, ash, flush, with_cpu=not args.no_cpu_baseline)
    other["c5_stream_1gpu"] = run_c5(torch, dev, ash)
    return dict(ms=ms, value=value, kms=kms, e2e_ms=e2e_ms, h2d=h2d, d2h=d2h, clocks=clk.summary(),
                sweep=sweep, other=other, launches=launches)


def run_other_configs(torch, dev, ash, flush, with_cpu: bool):
    """configs[2] (voxelize 20M sphere points at 5 mm) and configs[3] (block
    allocation for a 640x480 plane frame, 1.536M candidates): device time of
    the map path with CUDA events, and the CPU reference algorithm (oracle
    port) on a bounded sample beside it."""
    from paper_2110_00511_b200.workloads import sphere_points
    from oracle import ash_oracle as O
    stream = torch.cuda.current_stream(dev)
    out = {}
    pts_np = sphere_points(20_000_000, seed=0)
    pts = torch.from_numpy(pts_np).to(dev)
    ts = []
    for i in range(6):
        l2_flush(torch, flush)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        coords, sel = ash.voxel_downsample(pts, 0.005, device=dev)
        b.record(stream)
        torch.cuda.synchronize()
        if i:
            ts.append(a.elapsed_time(b))
    ms = statistics.median(ts)
    c3 = {"workload": "configs[2]: voxel_downsample of 20M unit-sphere points (float64) at 5 mm",
          "voxels": int(coords.shape[0]), "ms": round(ms, 3), "mpts_per_s": round(20e6 / ms / 1e3, 1),
          "note": "includes the count read-back (one 8-byte sync) that sizes the outputs"}
    if with_cpu:
        smp = pts_np[:2_000_000]
        t0 = time.perf_counter()
        O.voxel_downsample(smp, 0.005)
        c3["cpu_baseline"] = {"mpts_per_s": round(2.0 / (time.perf_counter() - t0), 3), "cores": 1,
                              "kind": "port", "sample": "first 2M points of the same cloud"}
    out["c3_voxelize"] = c3
    cam = O.scaled_camera(640, 480)
    depth = O.plane_depth(cam, 1.0)
    frames = []
    for f in range(10):
        pose = np.eye(4)
        pose[0, 3] = 0.02 * f
        frames.append(O.candidate_blocks(depth, cam, pose, 0.0058 * 8, 0.04))
    frames_d = [torch.from_numpy(c).to(dev) for c in frames]
    gm = ash.HashMap(100_000, 3, [((8, 8, 8, 2), np.float32)], device=dev)
    ts = []
    for rep in range(2):
        gm.clear()
        for c in frames_d:
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            ash.allocate_blocks(gm, c)
            b.record(stream)
            torch.cuda.synchronize()
            if rep:
                ts.append(a.elapsed_time(b))
    ms = statistics.median(ts)
    c4 = {"workload": "configs[3]: allocate_blocks map calls (local activate, global activate + find, "
                      "local value scatter), 640x480 plane frames, 1.536M candidates each, 10 frames",
          "blocks": gm.size, "ms_per_frame": round(ms, 3),
          "mcand_per_s": round(len(frames[0]) / ms / 1e3, 1),
          "note": "includes the host syncs of the boolean-mask gathers in the reference call sequence"}
    if with_cpu:
        og = O.OracleMap(100_000, 3, [((8, 8, 8, 2), np.float32)])
        t0 = time.perf_counter()
        O.allocate_blocks_map_calls(og, frames[0])
        c4["cpu_baseline"] = {"mcand_per_s": round(len(frames[0]) / (time.perf_counter() - t0) / 1e6, 3),
                              "cores": 1, "kind": "port", "sample": "first frame"}
    out["c4_allocate_blocks"] = c4
    # the same frames end to end from the depth image: fused candidate
    # generation + dedup on the device (§8(f) row 1), then the global activate
    depth_d = torch.from_numpy(depth).to(dev)
    grid = ash.BlockGrid(8, capacity=100_000, device=dev)
    ts = []
    for rep in range(2):
        grid.global_map.clear()
        for f in range(10):
            pose = np.eye(4)
            pose[0, 3] = 0.02 * f
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            grid.allocate_frame(depth_d, cam, pose)
            b.record(stream)
            torch.cuda.synchronize()
            if rep:
                ts.append(a.elapsed_time(b))
    assert grid.block_count == gm.size
    ms = statistics.median(ts)
    c4f = {"workload": "configs[3] from the depth image: fused candidate generation (ray mode, "
                       "fp64 in the reference's order) + dedup + global activate, 640x480 plane frames",
           "blocks": grid.block_count, "ms_per_frame": round(ms, 3),
           "mcand_per_s": round(len(frames[0]) / ms / 1e3, 1),
           "note": "includes the one 8-byte count read-back that sizes the frame's block list"}
    if with_cpu:
        og = O.OracleMap(100_000, 3, [((8, 8, 8, 2), np.float32)])
        t0 = time.perf_counter()
        O.allocate_blocks_map_calls(og, O.candidate_blocks(depth, cam, np.eye(4), 0.0058 * 8, 0.04))
        c4f["cpu_baseline"] = {"mcand_per_s": round(len(frames[0]) / (time.perf_counter() - t0) / 1e6, 3),
                               "cores": 1, "kind": "port",
                               "sample": "first frame: candidate generation + map calls"}
    out["c4_frame_fused"] = c4f
    return out


C5_TOTAL = 400_000_000
C5_BATCH = 1 << 25


def run_c5(torch, dev, ash):
    """configs[4] on one GPU: the 400M-key map built by the mixed stream
    (each step inserts 2^25 new keys and finds 2^25 keys, half present),
    keys generated in HBM by the counter-based generator.  The N-GPU
    hash-partitioned run of the same stream is `bench.py --c5` under torchrun."""
    from paper_2110_00511_b200.workloads import c5_step_batches
    stream = torch.cuda.current_stream(dev)
    steps = -(-C5_TOTAL // C5_BATCH)
    m = ash.HashMap(C5_TOTAL, 3, [np.float32], device=dev)
    ms_ins, ms_find, ops = [], [], 0
    for s in range(steps):
        ins, q = c5_step_batches(s * C5_BATCH, min(C5_BATCH, C5_TOTAL - s * C5_BATCH), C5_TOTAL, device=dev)
        vals = torch.rand((len(ins), 1), dtype=torch.float32, device=dev)
        torch.cuda.synchronize()
        a, b, c = (torch.cuda.Event(enable_timing=True) for _ in range(3))
        a.record(stream)
        r = m.insert(ins, vals)
        b.record(stream)
        f = m.find(q)
        c.record(stream)
        torch.cuda.synchronize()
        ms_ins.append(a.elapsed_time(b))
        ms_find.append(b.elapsed_time(c))
        ops += 2 * len(ins)
        assert bool(r.masks.all())
        hits = int(f.masks.sum())
        assert hits == len(q) // 2, hits
        del ins, q, vals, r, f
    assert m.size == C5_TOTAL
    tot = sum(ms_ins) + sum(ms_find)
    out = {"workload": "configs[4] at N=1: 400M-key map built by a mixed stream, 12 steps of "
                       "2^25 inserts (new keys, f32[1] values) + 2^25 finds (50% present)",
           "keys": C5_TOTAL, "ms_total": round(tot, 2), "mops": round(ops / tot / 1e3, 1),
           "insert_ms_first_last": [round(ms_ins[0], 3), round(ms_ins[-2], 3)],
           "find_ms_first_last": [round(ms_find[0], 3), round(ms_find[-2], 3)],
           "note": "table 9.6 GB (600M 16-byte slots); the map grows from 0 to 400M keys; "
                   "key generation and value fill excluded; no CPU baseline (400M is infeasible "
                   "for the reference)"}
    del m
    torch.cuda.empty_cache()
    return out


def run_sweep(torch, dev, ash, flush):
    """configs[1] sweep: rho in {0.1, 0.5, 1.0} x value f32[1] / f32[8];
    insert-only and find-only Mops/s (fresh map per trial)."""
    from paper_2110_00511_b200.workloads import int3_batch
    out = []
    stream = torch.cuda.current_stream(dev)
    for rho in (0.1, 0.5, 1.0):
        keys = torch.from_numpy(int3_batch(N_KEYS, rho, seed=0)).to(dev)
        for width in (1, 8):
            vals = torch.rand((N_KEYS, width), dtype=torch.float32, device=dev)
            m = ash.HashMap(CAPACITY, 3, [((width,), np.float32)], device=dev)
            ti, tf = [], []
            for trial in range(6):
                m.clear()
                l2_flush(torch, flush)
                a, b, c = (torch.cuda.Event(enable_timing=True) for _ in range(3))
                a.record(stream)
                m.insert(keys, vals)
                b.record(stream)
                l2_flush(torch, flush)
                b2 = torch.cuda.Event(enable_timing=True)
                b2.record(stream)
                m.find(keys)
                c.record(stream)
                torch.cuda.synchronize()
                if trial:
                    ti.append(a.elapsed_time(b))
                    tf.append(b2.elapsed_time(c))
            ims, fms = statistics.median(ti), statistics.median(tf)
            bw, _ = _peaks()
            ib = algorithmic_bytes("insert", rho, 4 * width) * N_KEYS
            fb = algorithmic_bytes("find", rho, 4 * width) * N_KEYS
            out.append({"rho": rho, "value": f"f32[{width}]",
                        "insert_mops": round(N_KEYS / ims / 1e3, 1),
                        "find_mops": round(N_KEYS / fms / 1e3, 1),
                        "insert_frac": round(ib / (ims / 1e3) / 1e9 / bw, 4),
                        "find_frac": round(fb / (fms / 1e3) / 1e9 / bw, 4)})
            del m
    return out


def _cpu_sample():
    """C2-shaped sample for the CPU arm: CPU_SAMPLE_KEYS keys per host core
    (uniqueness RHO, f32[1] values)."""
    import os as _os
    from paper_2110_00511_b200.workloads import int3_batch
    n = CPU_SAMPLE_KEYS * len(_os.sched_getaffinity(0))
    keys = int3_batch(n, RHO, seed=0)
    vals = np.random.default_rng(1).random((len(keys), 1), dtype=np.float32)
    return keys, vals


def cpu_baseline_sample():
    keys, vals = _cpu_sample()
    cpu = ShardedCpuReference(keys, vals)
    try:
        cpu.step()
        t = min(cpu.step() for _ in range(3))
    finally:
        cpu.close()
    # the reference's own reach: one process (its thread pool does not scale)
    one = keys[:CPU_SAMPLE_KEYS], vals[:CPU_SAMPLE_KEYS]
    t1 = min(cpu_reference_step(*one) for _ in range(2))
    return {"value": round(2 * cpu.n / t / 1e6, 4), "unit": UNIT, "cores": cpu.parts, "kind": "port",
            "sample": f"insert+find of {cpu.n:,} int3 keys (rho={RHO}, f32[1]) split by key hash over "
                      f"{cpu.parts} processes, each a fresh reference map of its shard (reference "
                      f"generic-backend algorithm via the numpy oracle port), best of 3",
            "single_process": {"value": round(2 * CPU_SAMPLE_KEYS / t1 / 1e6, 4), "cores": 1,
                               "sample": f"first {CPU_SAMPLE_KEYS:,} keys of the same sample, one map"}}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--partitioned", action="store_true",
                    help="force the hash-partitioned (torch.distributed) path even at N=1")
    ap.add_argument("--transport", default="peer", choices=["peer", "nccl"],
                    help="partitioned routing: peer-memory put/pull (symmetric memory) or NCCL all-to-all")
    ap.add_argument("--c5", action="store_true",
                    help="configs[4]: the 400M-key partitioned map built by the mixed stream (strong scaling)")
    ap.add_argument("--profile", action="store_true",
                    help="timed steps only (no sweep / e2e / cpu leg): for ncu captures")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))

    if args.impl == "reference":
        run_reference(args, rank, world)
        return

    import torch
    if world > 1 or args.partitioned or args.c5:
        from paper_2110_00511_b200 import partitioned
        partitioned.bench_main(args, rank, world)
        return
    dev = torch.device("cuda", int(os.environ.get("LOCAL_RANK", "0")))
    torch.cuda.set_device(dev)
    if args.profile:
        args.no_cpu_baseline = True
    res = gpu_single(args, torch, dev)
    bw, peak_kind = _peaks()
    kms = res["kms"]
    # dominant kernel and its roofline (algorithmic bytes per launch)
    per_kernel_bytes = {
        # key, probed sector, scratch idx+mask; each winner's CAS writes its slot sector
        "claim": (12 + 32 + 5) * N_KEYS + RHO * 32 * N_KEYS,
        # scratch in + out; winner key row, value read + write (the slot was written by the claim)
        "commit": (5 + 5) * N_KEYS + RHO * (12 + 2 * 4) * N_KEYS,
        "find": algorithmic_bytes("find", RHO, 4) * N_KEYS,
        "tile_scan": 4 * 2 * (N_KEYS / 2048),
    }
    dom = max(kms, key=kms.get)
    achieved = per_kernel_bytes[dom] / (kms[dom] / 1e3) / 1e9
    traffic, traffic_src = _profiled_traffic(f"k_{dom}")
    cpu = None if args.no_cpu_baseline else cpu_baseline_sample()
    line = {
        "metric": METRIC, "value": round(res["value"], 2), "unit": UNIT, "n_gpus": 1,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(res["ms"], 4),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "int32",
        "data": "synthetic",
        "config": {"workload": "configs[1]: 10M int3 keys, uniqueness 0.5, value f32[1]; "
                               "insert into a fresh capacity-10M map, then find the same keys",
                   "keys": N_KEYS, "uniqueness": RHO, "capacity": CAPACITY, "value": "f32[1]",
                   "l2": "flushed between steps (256 MB write); working set > L2",
                   "construction": "excluded (HashMap.clear before each step)"},
        "roofline": {"bound": "hbm", "kernel": f"k_{dom}", "achieved": round(achieved, 1),
                     "peak": bw, "peak_kind": peak_kind, "unit": "GB/s",
                     "frac": round(achieved / bw, 4), "traffic": traffic,
                     "traffic_source": traffic_src,
                     "algorithmic_bytes_per_launch": int(per_kernel_bytes[dom]),
                     "kernel_ms": {k: round(v, 4) for k, v in kms.items()}},
        "op_roofline": {
            "insert_frac": round(algorithmic_bytes("insert", RHO, 4) * N_KEYS /
                                 ((kms["claim"] + kms["tile_scan"] + kms["commit"]) / 1e3) / 1e9 / bw, 4),
            "find_frac": round(per_kernel_bytes["find"] / (kms["find"] / 1e3) / 1e9 / bw, 4)},
        # the bound that actually binds a random probe: DRAM bandwidth at the
        # ~85 B the memory system moves per 32-byte probe (profiles/*_random_access.json)
        "random_access": _random_access(kms),
        "e2e": {"value": round(2 * N_KEYS / (res["e2e_ms"] / 1e3) / 1e6, 2), "unit": UNIT,
                "h2d_bytes_per_step": int(res["h2d"]), "d2h_bytes_per_step": int(res["d2h"])},
        "gpu_launches": res["launches"],  # libash kernels in the timed region (ash_launch_count)
        "clocks": res["clocks"],
        "sweep": res["sweep"],
        "other_configs": res["other"],
        "cpu_baseline": cpu,
    }
    print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
