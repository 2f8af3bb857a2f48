"""SCAN schedule timings (not product code): device time (CUDA events around
one execute_batch_dptr) of 2^20-tx bank SCAN batches (uniform / zipf 0.99,
first batch of a round and a later one) and of a 2^20 GET/SET cache SCAN batch
(configs[3]); median of 5.  Run from a repo root: python tools/scan_timing_probe.py"""
import os
import statistics
import sys

sys.path.insert(0, os.getcwd())
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1905_00661_b200 as hetm  # noqa: E402

n, W = 1 << 20, 1 << 27


def timed(d, fn, reps=5, clear=True):
    ex = torch.cuda.ExternalStream(d.stream_handle(0))
    out = []
    for _ in range(reps + 1):
        d.sync()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(ex)
        fn()
        e1.record(ex)
        d.sync()
        if clear:
            d.clear_round()
        out.append(e0.elapsed_time(e1))
    return statistics.median(out[1:])


d = hetm.GpuDevice(W, rs_gran_bytes=1024)
d.register_kernel(hetm.KERNEL_BANK)
d.upload(hetm.REPLICA_DEV, 0, np.full(W, 1000, np.uint64))
tk = torch.empty(n, dtype=torch.int64, device="cuda")
d.set_schedule(hetm.SCHED_SCAN)
for z in (0.0, 0.99):
    b = torch.from_numpy(hetm.gen_bank_batch(70, n, 0, W // 2, zipf=z).view(np.uint8)).cuda()
    first = timed(d, lambda: d.execute_batch_dptr(hetm.KERNEL_BANK, b.data_ptr(), n, tk.data_ptr()))
    later = timed(d, lambda: d.execute_batch_dptr(hetm.KERNEL_BANK, b.data_ptr(), n, tk.data_ptr()), clear=False)
    print(f"bank SCAN zipf {z:4.2f}: first batch of a round {first:.4f} ms, later batch {later:.4f} ms", flush=True)
d.close()
n_sets = 1 << 20
dc = hetm.GpuDevice(n_sets * hetm.CACHE_SET_WORDS, rs_gran_bytes=1024)
dc.register_kernel(hetm.KERNEL_CACHE)
dc.set_cache_geometry(0, n_sets)
cb = torch.from_numpy(hetm.gen_cache_batch(7, n, 4 << 20, 0.5, 900, 1).view(np.uint8)).cuda()
ck = torch.empty(n, dtype=torch.int64, device="cuda")
t = timed(dc, lambda: dc.execute_batch_dptr(hetm.KERNEL_CACHE, cb.data_ptr(), n, ck.data_ptr()))
print(f"cache SCAN 90/10 zipf 0.5: {t:.4f} ms per 2^20", flush=True)
dc.close()
