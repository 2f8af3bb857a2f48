"""Kernel breakdown of one SCAN-schedule cache batch (not product code): CUPTI over
a 2^20-tx GET/SET 90/10 batch, zipf 0.5 over 4 M keys, 2^20 sets (cfg4 geometry)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from torch.profiler import ProfilerActivity, profile

import paper_1905_00661_b200 as hetm

B, n_sets = 1 << 20, 1 << 20
d = hetm.GpuDevice(n_sets * 64, rs_gran_bytes=1024)
d.register_kernel(hetm.KERNEL_CACHE)
d.set_schedule(hetm.SCHED_SCAN)
tk = torch.empty(B, dtype=torch.int64, device="cuda")
res = torch.empty(B * 40, dtype=torch.uint8, device="cuda")
warm = torch.from_numpy(hetm.gen_cache_batch(1, B, 1 << 22, 0.5, get_permille=0, part=1).view(np.uint8)).cuda()
d.execute_batch_dptr(hetm.KERNEL_CACHE, warm.data_ptr(), B, tk.data_ptr(), 0, res.data_ptr())
ALPHA = float(sys.argv[1]) if len(sys.argv) > 1 else 0.5
b = torch.from_numpy(hetm.gen_cache_batch(10, B, 1 << 22, ALPHA, get_permille=900, part=1).view(np.uint8)).cuda()
for _ in range(2):
    d.execute_batch_dptr(hetm.KERNEL_CACHE, b.data_ptr(), B, tk.data_ptr(), 0, res.data_ptr())
d.sync()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    d.execute_batch_dptr(hetm.KERNEL_CACHE, b.data_ptr(), B, tk.data_ptr(), 0, res.data_ptr())
    d.sync()
tot = 0.0
for e in prof.events():
    if e.device_type == torch.autograd.DeviceType.CUDA:
        tot += e.device_time
        print(f"  {e.device_time:8.1f} us  {e.name[:90]}")
print(f"  total {tot:.1f} us")
