"""Stripe-lock bank kernel across skew (not product code): device-pointer batches
of 2^20 transactions on the 1 GiB STMR, zipf alpha in a sweep, OPTIMISTIC
(stripe kernel) vs SCAN: ms per batch (handle timing brackets, mean of 8
batches after 2 warm-ups) and the optimistic kernel's aborted attempts per
transaction — the signal AUTO's abort feedback judges (capi.cu
kAutoAbortRatio)."""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_1905_00661_b200 as hetm

W, n = 1 << 27, 1 << 20
d = hetm.GpuDevice(W, rs_gran_bytes=1024)
d.register_kernel(hetm.KERNEL_BANK)
d.upload(hetm.REPLICA_DEV, 0, np.full(W, 1000, np.uint64))
tk = torch.empty(n, dtype=torch.int64, device="cuda")
print(f"stripe bits (HETM_STRIPE_BITS) {os.environ.get('HETM_STRIPE_BITS', '24 (default)')}")
for alpha in (0.0, 0.3, 0.4, 0.5, 0.6, 0.7):
    bt = [torch.from_numpy(hetm.gen_bank_batch(900 + k, n, 0, W, zipf=alpha).view(np.uint8)).cuda() for k in range(2)]
    row = [f"alpha {alpha:.1f}"]
    for name, sched in (("optimistic", hetm.SCHED_OPTIMISTIC), ("scan", hetm.SCHED_SCAN)):
        d.set_schedule(sched)
        ms, ab, rt = [], [], []
        for k in range(10):
            d.clear_round()
            d.timing(0)
            d.set_timing(True)
            d.execute_batch_dptr(hetm.KERNEL_BANK, bt[k % 2].data_ptr(), n, tk.data_ptr())
            d.sync()
            t, c = d.timing(0)
            d.set_timing(False)
            _, st = d.read_counters()
            if k >= 2:
                ms.append(t / max(c, 1))
                ab.append(st.aborts / n)
                rt.append(st.retried / n)
        row.append(f"{name} {statistics.mean(ms):.3f} ms" + (f" aborts/tx {statistics.mean(ab):.4f} retried/tx {statistics.mean(rt):.5f}" if name == "optimistic" else ""))
    print("  ".join(row), flush=True)
