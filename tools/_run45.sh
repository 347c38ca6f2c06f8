set -u
timeout 300 python tools/exp_host_cost.py 100000 2>&1 | head -1
timeout 300 python tools/exp_dedup.py c4 8 2>&1 | grep c4
timeout 300 python -c "
import sys; sys.path.insert(0,'.')
import torch
from paper_2110_00511_b200.hashmap import _stream_handle
d=torch.device('cuda',0)
s=torch.cuda.Stream()
assert _stream_handle(d)==torch.cuda.current_stream(d).cuda_stream
with torch.cuda.stream(s):
    assert _stream_handle(d)==s.cuda_stream
print('stream handle ok')
"
