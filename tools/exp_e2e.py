"""e2e (host in / host out) pipeline experiment on the GPU box: chunk size
sweep for HashMap insert+find of 10M pinned int3 keys, plus raw PCIe copy
rates for reference."""
import sys, time
sys.path.insert(0, ".")
import numpy as np
import torch
import paper_2110_00511_b200 as ash
from paper_2110_00511_b200.workloads import int3_batch

dev = torch.device("cuda:0")
N = 10_000_000
keys_h = torch.from_numpy(int3_batch(N, 0.5, seed=0)).pin_memory()
vals_h = torch.from_numpy(np.random.default_rng(1).random((N, 1), dtype=np.float32)).pin_memory()
buf = torch.empty(N * 3, dtype=torch.int32, device=dev)
hbuf = torch.empty(N * 3, dtype=torch.int32, pin_memory=True)
for name, fn in (("h2d 120MB", lambda: buf.copy_(keys_h.view(-1), non_blocking=True)),
                 ("d2h 120MB", lambda: hbuf.copy_(buf, non_blocking=True))):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(10):
        fn()
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t0) / 10
    print(f"{name}: {dt*1e3:.3f} ms  {120e6/dt/1e9:.1f} GB/s")
m = ash.HashMap(N, 3, [np.float32], device=dev)
for chunk in [int(c) for c in (sys.argv[1:] or ["2097152", "1048576", "524288", "262144"])]:
    ash.HashMap.PIPELINE_CHUNK = chunk
    ts, ti, tf = [], [], []
    for i in range(8):
        m.clear()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        r = m.insert(keys_h, vals_h)
        t1 = time.perf_counter()
        f = m.find(keys_h)
        t2 = time.perf_counter()
        if i >= 3:
            ts.append(t2 - t0); ti.append(t1 - t0); tf.append(t2 - t1)
    assert int(r.masks.sum()) == N // 2 and bool(f.masks.all())
    ms = 1e3 * sum(ts) / len(ts)
    print(f"chunk={chunk}: step {ms:.3f} ms  insert {1e3*sum(ti)/len(ti):.3f}  find {1e3*sum(tf)/len(tf):.3f}"
          f"  e2e {2*N/ms/1e3:.1f} Mops/s")

# floor: the same chunked copies with no kernels (H2D keys+vals, D2H idx+mask)
def copies_only(with_vals):
    c = 1 << 20
    h2d, d2h = torch.cuda.Stream(), torch.cuda.Stream()
    kd = torch.empty((N, 3), dtype=torch.int32, device=dev)
    vd = torch.empty((N, 1), dtype=torch.float32, device=dev)
    ih = torch.empty(N, dtype=torch.int32, pin_memory=True)
    mh = torch.empty(N, dtype=torch.uint8, pin_memory=True)
    idd = torch.zeros(N, dtype=torch.int32, device=dev)
    md = torch.zeros(N, dtype=torch.uint8, device=dev)
    s = torch.cuda.current_stream()
    for a in range(0, N, c):
        b = min(N, a + c)
        with torch.cuda.stream(h2d):
            kd[a:b].copy_(keys_h[a:b], non_blocking=True)
            if with_vals:
                vd[a:b].copy_(vals_h[a:b], non_blocking=True)
        d2h.wait_stream(h2d)
        with torch.cuda.stream(d2h):
            ih[a:b].copy_(idd[a:b], non_blocking=True)
            mh[a:b].copy_(md[a:b], non_blocking=True)
    d2h.synchronize()

for _ in range(3):
    copies_only(True); copies_only(False)
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(5):
    copies_only(True)
    copies_only(False)
torch.cuda.synchronize()
print(f"copies only (insert-like + find-like): {(time.perf_counter() - t0) / 5 * 1e3:.3f} ms per step")

def h2d_only():
    c = 1 << 20
    h2d = torch.cuda.Stream()
    kd = torch.empty((N, 3), dtype=torch.int32, device=dev)
    vd = torch.empty((N, 1), dtype=torch.float32, device=dev)
    for a in range(0, N, c):
        b = min(N, a + c)
        with torch.cuda.stream(h2d):
            kd[a:b].copy_(keys_h[a:b], non_blocking=True)
            vd[a:b].copy_(vals_h[a:b], non_blocking=True)
    for a in range(0, N, c):
        b = min(N, a + c)
        with torch.cuda.stream(h2d):
            kd[a:b].copy_(keys_h[a:b], non_blocking=True)
    h2d.synchronize()

for _ in range(3):
    h2d_only()
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(5):
    h2d_only()
torch.cuda.synchronize()
print(f"chunked H2D only (280 MB): {(time.perf_counter() - t0) / 5 * 1e3:.3f} ms per step")
