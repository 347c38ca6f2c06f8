"""PCIe copy rates on the GPU box (pinned host memory): H2D by stream count
and chunk size, and H2D + D2H at once (the e2e pipeline overlaps them)."""
import torch, time
dev = torch.device("cuda:0")
N = 120_000_000 // 4
h = torch.empty(N, dtype=torch.int32).pin_memory()
d = torch.empty(N, dtype=torch.int32, device=dev)
def run(k, chunk):
    streams = [torch.cuda.Stream() for _ in range(k)]
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for rep in range(5):
        for i, a in enumerate(range(0, N, chunk)):
            s = streams[i % k]
            with torch.cuda.stream(s):
                d[a:a+chunk].copy_(h[a:a+chunk], non_blocking=True)
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t0) / 5
    print(f"streams={k} chunk={chunk*4/1e6:.0f}MB: {120e6/dt/1e9:.1f} GB/s", flush=True)
for k in (1, 2, 4):
    for chunk in (N, 1 << 22, 1 << 20):
        run(k, chunk)
# duplex: H2D and D2H at once
hb = torch.empty(N, dtype=torch.int32).pin_memory()
d2 = torch.empty(N, dtype=torch.int32, device=dev)
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
torch.cuda.synchronize(); t0 = time.perf_counter()
for _ in range(5):
    with torch.cuda.stream(s1): d.copy_(h, non_blocking=True)
    with torch.cuda.stream(s2): hb.copy_(d2, non_blocking=True)
torch.cuda.synchronize(); dt = (time.perf_counter()-t0)/5
print(f"duplex: {120e6/dt/1e9:.1f} GB/s each way")
