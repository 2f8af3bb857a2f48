"""Where a BASELINE configs[2] round spends its time (host wall clock per call,
device synced after each): zipf(0.99) bank batch on the whole 1 GiB STMR, a
2^20-entry zipf(0.99) host log validated + applied, verdict, optimized
mergeAbortDevice (or merge_stage on a guard round), clear."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_1905_00661_b200 as hetm

B = 1 << 20
W = 1 << 27
d = hetm.GpuDevice(W, rs_gran_bytes=1024, log_capacity=B, merge_delta=True)
d.register_kernel(hetm.KERNEL_BANK)
d.upload(hetm.REPLICA_DEV, 0, np.full(W, 1000, np.uint64))
d.merge_commit(np.full(W, 1000, np.uint64))
d.merge_wait()
d.clear_round()
d.set_schedule(hetm.SCHED_SCAN)
bats = [torch.from_numpy(hetm.gen_bank_batch(60 + k, B, 0, W, zipf=0.99).view(np.uint8)).cuda() for k in range(2)]
logs = []
for r in range(10):
    lg = hetm.gen_host_log(70 + r, B // 2, 2, 8, 0, W, ts_base=(r + 1) << 32, zipf=0.99)
    logs.append(torch.from_numpy(lg.view(np.uint64).reshape(-1, 3).astype(np.int64)).cuda())
tk = torch.empty(B, dtype=torch.int64, device="cuda")


def t(label, fn, acc):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    r = fn()
    torch.cuda.synchronize()
    acc.setdefault(label, []).append((time.perf_counter() - t0) * 1e3)
    return r


acc = {}
for r in range(10):
    t("batch", lambda: d.execute_batch_dptr(hetm.KERNEL_BANK, bats[r % 2].data_ptr(), B, tk.data_ptr()), acc)
    guard = r % 4 == 3
    if not guard:
        t("validate", lambda: d.validate_dptr(logs[r].data_ptr(), B, hetm.APPLY | hetm.RETAIN), acc)
    c = t("verdict", d.round_verdict, acc)
    if c:
        t("abort", lambda: d.merge_abort_device(None, optimized=True), acc)
    else:
        t("stage", d.merge_stage, acc)
    t("clear", d.clear_round, acc)
for k, v in acc.items():
    print(f"{k:10s} n={len(v):2d} median {np.median(v):8.3f} ms  max {max(v):8.3f} ms  first {v[0]:8.3f}")
