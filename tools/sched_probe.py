"""Bank batch schedules across skew (not product code): OPTIMISTIC vs SCAN
time per 2^20-tx batch (isolated launch bracketed by the handle's timing
events, and pipelined: 10 batches back to back between two events) on the 1 GiB STMR for zipf alpha in a sweep,
next to the AUTO estimator's predicted chain (capi.cu bank_batch_hot:
hottest account count among 4096 sampled transactions x n / 4096).

    python tools/sched_probe.py [log2 n]
"""
import json
import os
import statistics
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_1905_00661_b200 as hetm

n = 1 << (int(sys.argv[1]) if len(sys.argv) > 1 else 20)
W = 1 << 27
d = hetm.GpuDevice(W, rs_gran_bytes=1024)
d.register_kernel(hetm.KERNEL_BANK)
d.upload(hetm.REPLICA_DEV, 0, np.full(W, 1000, np.uint64))
tickets = torch.empty(n, dtype=torch.int64, device="cuda")


def est_chain(txs):  # capi.cu bank_batch_hot: 32 evenly spaced blocks of 128 transactions
    per = min(128, n // 32)
    acc = np.concatenate([txs["acct"][b * (n // 32): b * (n // 32) + per] for b in range(32)]).reshape(-1)
    _, c = np.unique(acc, return_counts=True)
    return int(c.max()) * n // (32 * per)


def timed(sched, batch, reps):
    d.set_schedule(sched)
    ms = []
    for rep in range(reps + 1):
        d.set_timing(True)
        d.execute_batch_dptr(hetm.KERNEL_BANK, batch.data_ptr(), n, tickets.data_ptr())
        d.sync()
        t, _ = d.timing(0)
        d.set_timing(False)
        _, st = d.read_counters()
        d.clear_round()
        if rep:
            ms.append(t)
    return statistics.median(ms), st.aborts


ex = torch.cuda.ExternalStream(d.stream_handle(0))


def pipelined(sched, batch, k):
    """k batches back to back on the exec stream (host runs ahead, as in a
    round with several batches): device time per batch between two events."""
    d.set_schedule(sched)
    d.execute_batch_dptr(hetm.KERNEL_BANK, batch.data_ptr(), n, tickets.data_ptr())  # warm (graph capture)
    d.sync()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(ex)
    h0 = time.perf_counter()
    for _ in range(k):
        d.execute_batch_dptr(hetm.KERNEL_BANK, batch.data_ptr(), n, tickets.data_ptr())
    host_us = (time.perf_counter() - h0) * 1e6 / k
    e1.record(ex)
    d.sync()
    d.clear_round()
    return e0.elapsed_time(e1) / k, host_us


out = []
for alpha in [0.0, 0.5, 0.6, 0.7, 0.75, 0.8, 0.9, 0.99]:
    txs = hetm.gen_bank_batch(70, n, 0, W, zipf=alpha)
    b = torch.from_numpy(txs.view(np.uint8)).cuda()
    scan_ms, _ = timed(hetm.SCHED_SCAN, b, 3)
    opt_ms, ab = timed(hetm.SCHED_OPTIMISTIC, b, 1 if alpha >= 0.8 else 3)
    scan_pipe, scan_host_us = pipelined(hetm.SCHED_SCAN, b, 10)
    opt_pipe = pipelined(hetm.SCHED_OPTIMISTIC, b, 10)[0] if alpha <= 0.6 else None
    row = {"alpha": alpha, "n": n, "est_chain": est_chain(txs), "optimistic_ms": opt_ms, "optimistic_aborts": ab,
           "scan_ms": scan_ms, "scan_tx_per_s": n / scan_ms * 1e3, "auto_picks_scan": est_chain(txs) >= 768,
           "pipelined_scan_ms": scan_pipe, "pipelined_scan_tx_per_s": n / scan_pipe * 1e3,
           "pipelined_optimistic_ms": opt_pipe, "scan_host_enqueue_us": scan_host_us}
    out.append(row)
    print(json.dumps(row), flush=True)
