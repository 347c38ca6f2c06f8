"""configs[4] kernel breakdown on the GPU box: the 400M-key mixed stream of
bench.run_c5, meant to run under an ncu launch list, e.g.
  ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
      -k regex:"k_(claim|commit|tile|find)" -s 30 -c 10 python tools/exp_c5.py"""
import sys
sys.path.insert(0, ".")
import numpy as np
import torch
import paper_2110_00511_b200 as ash
from paper_2110_00511_b200.workloads import c5_step_batches

dev = torch.device("cuda:0")
TOTAL, BATCH = 400_000_000, 1 << 25
m = ash.HashMap(TOTAL, 3, [np.float32], device=dev)
for s in range(-(-TOTAL // BATCH)):
    ins, q = c5_step_batches(s * BATCH, min(BATCH, TOTAL - s * BATCH), TOTAL, device=dev)
    vals = torch.rand((len(ins), 1), dtype=torch.float32, device=dev)
    m.insert(ins, vals)
    m.find(q)
    torch.cuda.synchronize()
print("size", m.size)
