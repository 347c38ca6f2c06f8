import sys, time
sys.path.insert(0, ".")
import numpy as np, torch
import paper_2110_00511_b200 as ash
from paper_2110_00511_b200.workloads import int3_batch
for n in [int(x) for x in sys.argv[1:]]:
    keys = torch.from_numpy(int3_batch(n, 0.5, seed=1)).cuda()
    m = ash.HashMap(n, 3, device="cuda")
    torch.cuda.synchronize()
    t0 = time.time()
    r = m.insert(keys)
    torch.cuda.synchronize()
    print(n, "insert ok", time.time() - t0, int(r.masks.sum()), flush=True)
    f = m.find(keys)
    print(n, "find", bool(f.masks.all()), flush=True)
