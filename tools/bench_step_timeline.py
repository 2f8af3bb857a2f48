"""GPU timeline of bench.py's device step as it runs today (not product code):
execute_batch_dptr (2^20 bank tx) -> validate_dptr APPLY|RETAIN (2^20 entries)
-> merge_stage -> async clear, 12 steps back to back under CUPTI; prints the
ops (kernels, memsets, copies) of two steps with their start offsets, durations
and the idle gap before each."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from torch.profiler import ProfilerActivity, profile

import paper_1905_00661_b200 as hetm

W, B, L = 1 << 27, 1 << 20, 1 << 20
dev = hetm.GpuDevice(W, rs_gran_bytes=1024, log_capacity=L, merge_delta=True)
dev.register_kernel(hetm.KERNEL_BANK)
init = np.full(W, 1000, np.uint64)
dev.upload(hetm.REPLICA_DEV, 0, init)
host = hetm.PinnedArray((W,), np.uint64)
host.array[:] = init
dev.merge_commit(host.array)
dev.merge_wait()
dev.clear_round()
s_exec = dev.stream_handle(0)
s_val = dev.stream_handle(2)
txs = [torch.from_numpy(hetm.gen_bank_batch(100 + k, B, 0, W // 2).view(np.uint8)).cuda() for k in range(4)]
base_log = hetm.gen_host_log(200, L // 2, 2, 8, W // 2, W // 2, ts_base=0)
base_t = torch.from_numpy(base_log.view(np.uint64).reshape(-1, 3).astype(np.int64)).cuda()
logs = []
for k in range(16):
    t = base_t.clone()
    t[:, 2] += k * (L // 2) + 1
    logs.append(t)
tk = torch.empty(B, dtype=torch.int64, device="cuda")


def step(j):
    dev.execute_batch_dptr(hetm.KERNEL_BANK, txs[j % 4].data_ptr(), B, tk.data_ptr(), s_exec)
    dev.validate_dptr(logs[j].data_ptr(), L, hetm.APPLY | hetm.RETAIN, s_val)
    dev.merge_stage()
    dev.clear_round(asynchronous=True)


for j in range(3):
    step(j)
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    for j in range(3, 15):
        step(j)
    torch.cuda.synchronize()
ev = sorted([e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA],
            key=lambda e: e.time_range.start)
bank = [e for e in ev if "bank_batch_kernel" in e.name]
t0, t1 = bank[4].time_range.start, bank[8].time_range.start  # four full steps
prev_end = None
for e in ev:
    if t0 <= e.time_range.start < bank[6].time_range.start:
        gap = "" if prev_end is None else f" gap {e.time_range.start - prev_end:6.1f}"
        print(f"{e.time_range.start - t0:8.1f} +{e.time_range.end - e.time_range.start:7.1f}{gap}  {e.name[:70]}")
        prev_end = max(prev_end or 0, e.time_range.end)
print(f"per step: {(t1 - t0) / 4:.1f} us")
