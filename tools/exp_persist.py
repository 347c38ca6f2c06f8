"""configs[2] with the dedup workspace prefix marked L2-persisting (GPU box):
cudaLimitPersistingL2CacheSize + a stream access-policy window over the
workspace slots during voxel_downsample, against the default; results
compared."""
import statistics
import sys

sys.path.insert(0, ".")
import torch
from cuda.bindings import runtime as rt

import paper_2110_00511_b200 as ash
from paper_2110_00511_b200.geometry import _VoxelWorkspace
from paper_2110_00511_b200.workloads import sphere_points

dev = torch.device("cuda:0")
pts = torch.from_numpy(sphere_points(20_000_000, seed=0)).to(dev)
stream = torch.cuda.current_stream(dev)
flush = torch.zeros(64 * 1024 * 1024, dtype=torch.float32, device=dev)
ref = ash.voxel_downsample(pts, 0.005, device=dev)
ws = _VoxelWorkspace.get(dev)
prop = rt.cudaGetDeviceProperties(0)[1]
print("persisting max", prop.persistingL2CacheMaxSize, "window max", prop.accessPolicyMaxWindowSize, flush=True)


def set_window(nbytes):
    attr = rt.cudaStreamAttrValue()
    w = attr.accessPolicyWindow
    w.base_ptr = ws.slots.data_ptr()
    w.num_bytes = nbytes
    w.hitRatio = 1.0 if nbytes else 0.0
    w.hitProp = rt.cudaAccessProperty.cudaAccessPropertyPersisting
    w.missProp = rt.cudaAccessProperty.cudaAccessPropertyStreaming
    err, = rt.cudaStreamSetAttribute(stream.cuda_stream, rt.cudaStreamAttrID.cudaLaunchAttributeAccessPolicyWindow, attr)
    assert err == rt.cudaError_t.cudaSuccess, err


def run(persist):
    ts = []
    for i in range(12):
        flush.add_(1)
        if persist:
            set_window(min(persist, prop.accessPolicyMaxWindowSize))
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        c, s = ash.voxel_downsample(pts, 0.005, device=dev)
        b.record(stream)
        torch.cuda.synchronize()
        if persist:
            set_window(0)
            rt.cudaCtxResetPersistingL2Cache()
        if i >= 2:
            ts.append(a.elapsed_time(b))
        same = torch.equal(c, ref[0]) and torch.equal(s, ref[1])
    return statistics.median(ts), same


for limit_mb in (0, 32, 48, 64):
    if limit_mb:
        rt.cudaDeviceSetLimit(rt.cudaLimit.cudaLimitPersistingL2CacheSize, min(limit_mb << 20, prop.persistingL2CacheMaxSize))
    ms, same = run(ws.struct.n_slots * 16 if limit_mb else 0)
    print(f"persist limit {limit_mb} MB (window {ws.struct.n_slots * 16 >> 20} MB): {ms:.4f} ms  same={same}", flush=True)
