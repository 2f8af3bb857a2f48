"""Side measurements of BASELINE configs[2] (zipf) and configs[3] (cache) on one
B200 (not the bench line; results go to profiles/).  Device-resident inputs,
CUDA-event kernel times from the library's own brackets."""
import json
import os
import statistics
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_1905_00661_b200 as hetm


def timed_batches(d, kernel, batches, tickets, results=None, reps=3):
    ms, ab = [], []
    for rep in range(reps + 1):
        for b in batches:
            d.set_timing(True)
            d.execute_batch_dptr(kernel, b.data_ptr(), b.numel() // (56 if kernel == hetm.KERNEL_CACHE else 24),
                                 tickets.data_ptr(), 0, results.data_ptr() if results is not None else 0)
            d.sync()
            t, _ = d.timing(0)
            d.set_timing(False)
            _, st = d.read_counters()
            d.clear_round()
            if rep:
                ms.append(t)
                ab.append(st.aborts)
    return (statistics.median(ms), statistics.median(ab)) if ms else (None, None)


out = {}
B = 1 << 20
# configs[2]: zipf bank batches on the 1 GiB STMR
W = 1 << 27
d = hetm.GpuDevice(W, rs_gran_bytes=1024)
d.register_kernel(hetm.KERNEL_BANK)
d.upload(hetm.REPLICA_DEV, 0, np.full(W, 1000, np.uint64))
tickets = torch.empty(B, dtype=torch.int64, device="cuda")
for alpha in [0.0, 0.5, 0.8, 0.99]:
    bs = [torch.from_numpy(hetm.gen_bank_batch(50 + k, B, 0, W, zipf=alpha).view(np.uint8)).cuda() for k in range(2)]
    ms, ab = timed_batches(d, hetm.KERNEL_BANK, bs, tickets, reps=1 if alpha > 0.7 else 3)
    out[f"cfg3_bank_zipf{alpha}"] = {"batch_ms": ms, "tx_per_s": B / ms * 1e3, "aborts_per_batch": ab}
    print(f"cfg3 bank zipf {alpha}: {ms:.3f} ms/batch, {B / ms / 1e6:.3f} G tx/s, aborts {ab}", flush=True)
# rollback cost: one conflicting round (zipf host log) -> optimized mergeAbortDevice
host = np.full(W, 1000, np.uint64)
d.upload(hetm.REPLICA_DEV, 0, host)
d.merge_commit(host)  # shadow == round start
d.merge_wait()
d.clear_round(reset_ts=True)
txs = hetm.gen_bank_batch(77, B, 0, W, zipf=0.5)
r = d.execute_batch(hetm.KERNEL_BANK, txs, want_tickets=False)
log = hetm.gen_host_log(78, B // 2, 2, 8, 0, W, ts_base=1 << 40, zipf=0.99)
keep = [d.stream_chunk(c, src_thread=i) for i, c in enumerate(np.array_split(log, 8))]
assert d.round_verdict()
t = time.perf_counter()
ms = d.merge_abort_device(host, optimized=True)
rb = (time.perf_counter() - t) * 1e3
hetm.gen_host_log(78, B // 2, 2, 8, 0, W, ts_base=1 << 40, zipf=0.99)
o = np.argsort(log["ts"], kind="stable")
host[log["addr"][o]] = log["value"][o]
assert (d.download(hetm.REPLICA_DEV) == host).all(), "rollback != host replica"

out["cfg3_rollback_optimized_ms"] = rb
print(f"cfg3 optimized rollback (2^20-entry zipf log, 1 GiB STMR): {rb:.2f} ms host wall", flush=True)
del keep
d.close()

# configs[3]: cache, 2^20 sets x 8 ways (512 MiB of words)
n_sets = 1 << 20
W = n_sets * 64
d = hetm.GpuDevice(W, rs_gran_bytes=1024)
d.register_kernel(hetm.KERNEL_CACHE)
res = torch.empty(B * 40, dtype=torch.uint8, device="cuda")
warm = torch.from_numpy(hetm.gen_cache_batch(1, B, 1 << 22, 0.5, get_permille=0, part=1).view(np.uint8)).cuda()
timed_batches(d, hetm.KERNEL_CACHE, [warm], tickets, res, reps=0)
sched_names = {hetm.SCHED_AUTO: "", hetm.SCHED_OPTIMISTIC: "_optimistic", hetm.SCHED_SCAN: "_scan"}
for sched in [hetm.SCHED_AUTO, hetm.SCHED_OPTIMISTIC, hetm.SCHED_SCAN]:
    d.set_schedule(sched)
    for gp in [900, 999]:
        bs = [torch.from_numpy(hetm.gen_cache_batch(10 + k, B, 1 << 22, 0.5, get_permille=gp, part=1).view(np.uint8)).cuda()
              for k in range(2)]
        ms, ab = timed_batches(d, hetm.KERNEL_CACHE, bs, tickets, res)
        key = f"cfg4_cache_get{gp / 10:.1f}{sched_names[sched]}"
        out[key] = {"batch_ms": ms, "tx_per_s": B / ms * 1e3, "aborts_per_batch": ab}
        print(f"{key}: {ms:.3f} ms/batch, {B / ms / 1e6:.3f} G tx/s, aborts {ab}", flush=True)
print(json.dumps(out))
