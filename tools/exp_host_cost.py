"""Host cost of the public API per call (GPU box): wall time of back-to-back
insert + find pairs on a small batch (the GPU finishes each pair faster than
the host issues it), and a cProfile of the Python side."""
import cProfile
import pstats
import sys
import time

sys.path.insert(0, ".")
import numpy as np
import torch

import paper_2110_00511_b200 as ash
from paper_2110_00511_b200.workloads import int3_batch

dev = torch.device("cuda:0")
n = int(sys.argv[1]) if len(sys.argv) > 1 else 100_000
keys = torch.from_numpy(int3_batch(n, 0.5, seed=3)).to(dev)
vals = torch.rand((n, 1), device=dev)
m = ash.HashMap(2 * n, 3, [np.float32], device=dev)


def pair():
    m.clear()
    m.insert(keys, vals)
    m.find(keys)


for _ in range(50):
    pair()
torch.cuda.synchronize()
t0 = time.perf_counter()
R = 500
for _ in range(R):
    pair()
torch.cuda.synchronize()
print(f"n={n}: {(time.perf_counter() - t0) / R * 1e6:.1f} us per clear+insert+find (wall, back-to-back)")
pr = cProfile.Profile()
pr.enable()
for _ in range(200):
    pair()
torch.cuda.synchronize()
pr.disable()
st = pstats.Stats(pr)
st.sort_stats("tottime").print_stats(22)
