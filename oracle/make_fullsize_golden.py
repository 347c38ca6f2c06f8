"""Full-size golden digests written by running the REFERENCE itself.

Run in the build container (where /root/reference exists):

    python oracle/make_fullsize_golden.py            # C1, C2 (six points), C3

The configs[1] (10M keys) and configs[2] (20M points) outputs are too large
to commit as arrays, so this script records SHA-256 digests of the
reference's own outputs on BASELINE.json's exact inputs:

  * gen_keys (pkg/src/spatialhash/bench.py:25-48) at C1 and the three C2
    uniqueness points, seed 0 — pins ``workloads.gen_keys``;
  * C1 and the six C2 points (rho in {0.1, 0.5, 1.0} x f32[1] / f32[8]):
    ``HashMap(n, 3, [((w,), float32)])`` (capacity = batch length, as in
    bench.py:103-106), values ``default_rng(1).random((n, w), float32)``
    (bench.py:114-116), insert then find of the same keys: the indices and
    masks of both calls, the size, and the key / value rows 0..size-1;
  * C3: ``voxel_downsample`` of the 20M-point unit sphere at 5 mm
    (geometry.py:59-76): coords and selected.

``tests/test_fullsize_gpu.py`` hashes the CUDA map's outputs on the same
inputs and compares (bit-exact: with a fresh heap every index is exact).
The reference's wall times here are recorded for information only.
"""
from __future__ import annotations

import hashlib
import json
import sys
import time
from pathlib import Path

import numpy as np

REF = Path("/root/reference/pkg/src")
ROOT = Path(__file__).resolve().parent.parent
OUT = ROOT / "tests" / "golden" / "fullsize_sha.json"


def sha(a) -> str:
    a = np.ascontiguousarray(np.asarray(a))
    if a.dtype == np.bool_:
        a = a.view(np.uint8)
    return hashlib.sha256(a.tobytes()).hexdigest()


def map_digest(HashMap, keys, width):
    n = len(keys)
    vals = np.random.default_rng(1).random((n, width), dtype=np.float32)
    m = HashMap(n, 3, [((width,), np.float32)])
    t0 = time.perf_counter()
    r = m.insert(keys, vals)
    t1 = time.perf_counter()
    f = m.find(keys)
    t2 = time.perf_counter()
    s = m.size
    return {
        "n": n, "width": width, "size": int(s),
        "insert_indices": sha(r.indices.astype(np.int32)), "insert_masks": sha(r.masks),
        "find_indices": sha(f.indices.astype(np.int32)), "find_masks": sha(f.masks),
        "key_rows": sha(m.key_buffer[:s]), "value_rows": sha(m.value_buffer(0)[:s]),
        "ref_insert_s": round(t1 - t0, 3), "ref_find_s": round(t2 - t1, 3),
    }


def main():
    sys.path.insert(0, str(REF))
    from spatialhash import HashMap, voxel_downsample
    from spatialhash.bench import gen_keys
    out = {"source": "reference spatialhash (/root/reference/pkg/src), numpy " + np.__version__,
           "gen_keys": {}, "maps": {}, "c3": None}
    points = [("c1", 100_000, 0.5, (1,))] + [(f"c2_rho{r}", 10_000_000, r, (1, 8)) for r in (0.1, 0.5, 1.0)]
    for name, n, rho, widths in points:
        t0 = time.perf_counter()
        keys = gen_keys(n, rho, "int3", seed=0)
        out["gen_keys"][name] = {"n": n, "rho": rho, "seed": 0, "sha": sha(keys),
                                 "ref_gen_s": round(time.perf_counter() - t0, 2)}
        for w in widths:
            d = map_digest(HashMap, keys, w)
            out["maps"][f"{name}_f32x{w}"] = dict(rho=rho, **d)
            print(name, w, d, flush=True)
    rng = np.random.default_rng(0)
    pts = rng.normal(size=(20_000_000, 3))
    pts /= np.linalg.norm(pts, axis=1, keepdims=True)
    t0 = time.perf_counter()
    coords, sel = voxel_downsample(pts, 0.005)
    out["c3"] = {"n": len(pts), "voxel": 0.005, "voxels": int(len(sel)),
                 "coords": sha(coords.astype(np.int32)), "selected": sha(sel.astype(np.int64)),
                 "ref_s": round(time.perf_counter() - t0, 2)}
    print(out["c3"], flush=True)
    OUT.write_text(json.dumps(out, indent=1) + "\n")


if __name__ == "__main__":
    main()
