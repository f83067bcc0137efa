#!/bin/bash
# One-off probe of the GPU box: host cores/RAM, GPU memory, torch read bandwidth.
set -x
nproc; free -g; lscpu | head -20; nvidia-smi; nvidia-smi topo -m
python - <<'PY'
import torch, time
print(torch.cuda.get_device_name(0), torch.cuda.mem_get_info())
a = torch.empty(8*1024**3//8, dtype=torch.float64, device='cuda').normal_()
torch.cuda.synchronize()
for _ in range(3): s = a.sum()
e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(10): s = a.sum()
e1.record(); torch.cuda.synchronize()
print("sum read GB/s", 10*a.numel()*8/ (e0.elapsed_time(e1)/1e3)/1e9)
PY
