set -u
O=gpurun_out
timeout 600 python tools/exp_spec.py > $O/r02zq_spec.log 2>&1; echo rc=$?; cat $O/r02zq_spec.log | tail -15
for S in 1 0; do
ASH_SPEC=$S timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_claim\|k_commit\|k_tile --csv --log-file $O/r02zq_launch_s$S.csv python -c "
import sys; sys.path.insert(0,'.')
import numpy as np, torch, paper_2110_00511_b200 as ash
from paper_2110_00511_b200.workloads import gen_keys
N=10_000_000
k=torch.from_numpy(gen_keys(N,0.1,'int3',seed=0)).cuda(); v=torch.rand((N,1),device='cuda')
m=ash.HashMap(N,3,[np.float32],device='cuda')
for _ in range(3):
    m.clear(); m.insert(k,v)
torch.cuda.synchronize()
" > /dev/null 2>&1; echo ncu rc=$?
python tools/summarize_profiles.py $O/r02zq_launch_s$S.csv 2>&1 | head -12
done
