"""configs[2] voxelize on the GPU box: timing + launch list helper."""
import sys, time
sys.path.insert(0, ".")
import torch
import paper_2110_00511_b200 as ash
from paper_2110_00511_b200.workloads import sphere_points
dev = torch.device("cuda:0")
pts = torch.from_numpy(sphere_points(20_000_000, seed=0)).to(dev)
for i in range(5):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    c, s = ash.voxel_downsample(pts, 0.005, device=dev)
    b.record()
    torch.cuda.synchronize()
    print(i, round(a.elapsed_time(b), 3), c.shape[0])
# a denser call after a sparse one: the estimate-sized table overflows once
c2, s2 = ash.voxel_downsample(pts, 0.0005, device=dev)
print("dense", c2.shape[0])
c3, s3 = ash.voxel_downsample(pts, 0.005, device=dev)
print("sparse again", c3.shape[0], bool((c3 == c).all()))
