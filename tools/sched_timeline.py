"""Kernel breakdown of one SCAN-schedule bank batch (not product code): torch.profiler
(CUPTI) over a 2^20-tx batch on the 1 GiB STMR, uniform and zipf 0.99."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from torch.profiler import ProfilerActivity, profile

import paper_1905_00661_b200 as hetm

n, W = 1 << 20, 1 << 27
d = hetm.GpuDevice(W, rs_gran_bytes=1024)
d.register_kernel(hetm.KERNEL_BANK)
d.set_schedule(hetm.SCHED_SCAN)
d.upload(hetm.REPLICA_DEV, 0, np.full(W, 1000, np.uint64))
tk = torch.empty(n, dtype=torch.int64, device="cuda")
cases = [(0.0, False), (0.99, False)] + ([(0.0, True), (0.99, True)] if "--first" in sys.argv else [])
for alpha, first in cases:
    b = torch.from_numpy(hetm.gen_bank_batch(5, n, 0, W, zipf=alpha).view(np.uint8)).cuda()
    for _ in range(3):
        d.execute_batch_dptr(hetm.KERNEL_BANK, b.data_ptr(), n, tk.data_ptr())
    d.sync()
    if first:  # the first batch of a round (bitmaps just cleared)
        d.clear_round()
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        d.execute_batch_dptr(hetm.KERNEL_BANK, b.data_ptr(), n, tk.data_ptr())
        d.sync()
    d.clear_round()
    print(f"== alpha {alpha}{' (first batch of the round)' if first else ''}")
    ks = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
    if ks:
        t0 = min(e.time_range.start for e in ks)
        t1 = max(e.time_range.end for e in ks)
        print(f"  span first start -> last end: {t1 - t0:.1f} us over {len(ks)} GPU ops")
    tot = 0.0
    for e in prof.events():
        if e.device_type == torch.autograd.DeviceType.CUDA:
            tot += e.device_time
            print(f"  {e.device_time:8.1f} us  {e.name[:90]}")
    print(f"  total {tot:.1f} us")
