"""configs[3] per-frame host overhead breakdown (GPU box): wall time of
allocate_blocks vs the device time of its kernels, and the host time of each
Python step of blocks._allocate_fused (perf_counter, synchronised only at
the status read the real path does)."""
import ctypes
import statistics
import sys
import time

sys.path.insert(0, ".")
import numpy as np
import torch

import paper_2110_00511_b200 as ash
from oracle import ash_oracle as O
from paper_2110_00511_b200 import _lib, blocks
from paper_2110_00511_b200.geometry import _VoxelWorkspace
from paper_2110_00511_b200.hashmap import _stream_handle

dev = torch.device("cuda:0")
cam = O.scaled_camera(640, 480)
depth = O.plane_depth(cam, 1.0)
frames = []
for f in range(10):
    pose = np.eye(4)
    pose[0, 3] = 0.02 * f
    frames.append(torch.from_numpy(O.candidate_blocks(depth, cam, pose, 0.0058 * 8, 0.04)).to(dev))
gm = ash.HashMap(100_000, 3, [((8, 8, 8, 2), np.float32)], device=dev)
for c in frames:
    ash.allocate_blocks(gm, c)
torch.cuda.synchronize()

walls = []
for rep in range(3):
    for c in frames:
        t0 = time.perf_counter()
        ash.allocate_blocks(gm, c)
        torch.cuda.synchronize()
        walls.append((time.perf_counter() - t0) * 1e3)
print("wall ms/frame median", round(statistics.median(walls), 4))

steps = {}


def tick(name, t):
    now = time.perf_counter()
    steps.setdefault(name, []).append((now - t) * 1e6)
    return now


for rep in range(3):
    for coords in frames:
        t = time.perf_counter()
        coords = gm._check_keys(coords).contiguous()
        t = tick("check_keys", t)
        n = coords.shape[0]
        ws = _VoxelWorkspace.get(dev)
        with _VoxelWorkspace._lock, torch.cuda.device(dev), gm._guard.writing():
            t = tick("enter", t)
            gm._settle()
            ws.reserve(n)
            gm._ensure_scan(n)
            gm._reserve_slots(max(gm._capacity - gm._top_ub, 0))
            t = tick("reserve", t)
            out, gi, gmask, si, sm, st = ws.sequence_buffers(n)
            stream = _stream_handle(dev)
            t = tick("alloc", t)
            slots, probe = next(ws.attempts())
            ws.use(slots, probe)
            _lib.call("ash_allocate_blocks", gm._ptr(), ctypes.byref(ws.struct), coords.data_ptr(), n,
                      out.data_ptr(), gi.data_ptr(), gmask.data_ptr(), si.data_ptr(), sm.data_ptr(), st.data_ptr(),
                      int(ws.estimate <= blocks._SMALL_ACTIVATE), stream)
            t = tick("launch (C call)", t)
            vals = st.tolist()
            t = tick("status read (sync)", t)
            gm._top_ub = min(gm._capacity, gm._top_ub + vals[4])
            res = out[:vals[1]].clone(), gi[:vals[1]].clone()
            blocks.LocalBlockMap(res[0], res[1], n, dev)
            t = tick("tail", t)
for k, v in steps.items():
    print(f"{k:22s} {statistics.median(v):8.1f} us")
