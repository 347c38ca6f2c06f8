"""Check that the oracle port is a faithful stand-in for the reference CPU
path: same outputs and the same speed on the same input.

Run in the build container (needs /root/reference):
    python oracle/time_vs_reference.py [n_keys]

Recorded result (this container, 8-core Xeon, 2M keys, rho=0.5, f32[1],
insert+find, best of 3): reference 2.859 Mops/s, oracle 2.830 Mops/s,
identical indices and masks.
"""
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, "/root/reference/pkg/src")

from spatialhash import HashMap  # noqa: E402  (the reference)

from oracle.ash_oracle import OracleMap  # noqa: E402
from paper_2110_00511_b200.workloads import int3_batch  # noqa: E402


def main(n: int = 2_000_000):
    keys = int3_batch(n, 0.5, seed=0)
    vals = np.random.default_rng(1).random((n, 1), dtype=np.float32)
    for name, cls in (("reference", HashMap), ("oracle", OracleMap)):
        ts = []
        for _ in range(3):
            m = cls(n, 3, [np.float32])
            t0 = time.perf_counter()
            m.insert(keys, vals)
            m.find(keys)
            ts.append(time.perf_counter() - t0)
        print(f"{name:9s} best {min(ts):.3f} s  {2 * n / min(ts) / 1e6:.3f} Mops/s")
    a = HashMap(n, 3, [np.float32]).insert(keys, vals)
    b = OracleMap(n, 3, [np.float32]).insert(keys, vals)
    print("identical indices/masks:", np.array_equal(a.indices, b.indices) and np.array_equal(a.masks, b.masks))


if __name__ == "__main__":
    main(int(sys.argv[1]) if len(sys.argv) > 1 else 2_000_000)
