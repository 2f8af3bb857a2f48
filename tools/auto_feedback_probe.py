"""AUTO's abort feedback on host-buffer bank batches (not product code): 32 batches of
2^20 zipf-0.5 transactions on the 1 GiB STMR (the band AUTO's sample cannot flag),
AUTO vs forced OPTIMISTIC / SCAN: kernel ms per batch (sum over the pipelined pieces)."""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

import paper_1905_00661_b200 as hetm

W, n, K = 1 << 27, 1 << 20, 32
d = hetm.GpuDevice(W, rs_gran_bytes=1024)
d.register_kernel(hetm.KERNEL_BANK)
d.upload(hetm.REPLICA_DEV, 0, np.full(W, 1000, np.uint64))
batches = [hetm.gen_bank_batch(700 + k, n, 0, W, zipf=0.5) for k in range(4)]
for name, sched in [("optimistic", hetm.SCHED_OPTIMISTIC), ("scan", hetm.SCHED_SCAN), ("auto", hetm.SCHED_AUTO)]:
    d.set_schedule(sched)
    ms, scan_runs = [], 0
    for k in range(K):
        r = d.execute_batch(hetm.KERNEL_BANK, batches[k % 4])
        ms.append(r.kernel_ms)
        scan_runs += r.aborts == 0 and bool((np.diff(r.tickets.astype(np.int64)) == 1).all())
        d.clear_round()
    print(f"{name:10s} mean {statistics.mean(ms):.3f} ms  median {statistics.median(ms):.3f} ms  "
          f"batches run as SCAN {scan_runs}/{K}")
