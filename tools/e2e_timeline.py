"""GPU timeline of the bench's end-to-end round (not product code).

Runs the bench.py e2e loop (2^20-tx bank batch + 2^20-entry host log per
round, delta merge) under torch.profiler (CUPTI activity tracing sees every
kernel and copy of the process, including libhetm_b200.so's streams) and
prints, for two steady-state rounds, each GPU activity with its stream,
start and duration relative to the round start, plus the host phases.

    python tools/e2e_timeline.py [--out gpurun_out/e2e_trace.json]
"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import ctypes as C

import numpy as np
import torch
from torch.profiler import ProfilerActivity, profile, record_function

import paper_1905_00661_b200 as hetm

W, B, L = 1 << 27, 1 << 20, 1 << 20
out = sys.argv[sys.argv.index("--out") + 1] if "--out" in sys.argv else "gpurun_out/e2e_trace.json"
EARLY = "--early" in sys.argv
dev = hetm.GpuDevice(W, rs_gran_bytes=1024, log_capacity=L, merge_delta=True)
dev.register_kernel(hetm.KERNEL_BANK)
if "--optimistic" in sys.argv:
    dev.set_schedule(hetm.SCHED_OPTIMISTIC)
init = np.full(W, 1000, np.uint64)
dev.upload(hetm.REPLICA_DEV, 0, init)
host = hetm.PinnedArray((W,), np.uint64)
host.array[:] = init
dev.merge_commit(host.array)
dev.merge_wait()
dev.clear_round()
txs = [hetm.PinnedArray((B,), hetm.BANK_TX) for _ in range(2)]
for j, p in enumerate(txs):
    hetm.gen_bank_batch(555 + j, B, 0, W // 2, out=p.array)
steps = 6
logs = [hetm.PinnedArray((L,), hetm.LOG_ENTRY) for _ in range(steps)]
for j, p in enumerate(logs):
    hetm.gen_host_log(900 + j, L // 2, 2, 8, W // 2, W // 2, ts_base=10_000_000_000 + j * L, out=p.array)
tickets = hetm.PinnedArray((B,), np.uint64)
lib = hetm._lib.lib


def round_(j):
    st = hetm._lib.BatchStats()
    with record_function("H execute_batch"):
        hetm.check(lib.hetm_dev_execute_batch(dev.h, hetm.KERNEL_BANK, txs[j % 2].array.ctypes.data, 24, B,
                                              tickets.array.ctypes.data, C.byref(st)), dev.h)
    if EARLY:
        with record_function("H merge_prepare"):
            dev.merge_prepare(host.array)
    else:
        with record_function("H merge_wait"):
            dev.merge_wait()
    lg = logs[j].array
    with record_function("H stream_chunks"):
        for c in range(8):
            dev.stream_chunk(lg[c * (L // 8):(c + 1) * (L // 8)], src_thread=c, seq=c)
    with record_function("H verdict"):
        assert not dev.round_verdict()
    with record_function("H merge_commit"):
        dev.merge_commit(host.array)
    with record_function("H clear_round"):
        dev.clear_round()


for j in range(3):
    round_(j)
dev.merge_wait()
with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA]) as prof:
    t0 = time.perf_counter()
    for j in range(3, 6):
        with record_function(f"ROUND {j}"):
            round_(j)
    dev.merge_wait()
    wall = (time.perf_counter() - t0) * 1e3
os.makedirs(os.path.dirname(out) or ".", exist_ok=True)
prof.export_chrome_trace(out)
ev = json.load(open(out))["traceEvents"]
rounds = sorted([e for e in ev if e.get("name", "").startswith("ROUND ")], key=lambda e: e["ts"])
gpu = [e for e in ev if e.get("cat") in ("kernel", "gpu_memcpy", "gpu_memset") and "dur" in e]
host_ph = [e for e in ev if e.get("name", "").startswith("H ") and "dur" in e]
print(f"3 rounds wall {wall:.2f} ms ({wall / 3:.2f} ms/round)")
for r in rounds[:2]:
    r0, r1 = r["ts"], r["ts"] + r["dur"]
    print(f"== {r['name']}  {r['dur'] / 1e3:.3f} ms")
    for e in sorted(host_ph, key=lambda e: e["ts"]):
        if r0 <= e["ts"] < r1:
            print(f"   host  {(e['ts'] - r0) / 1e3:7.3f} +{e['dur'] / 1e3:6.3f}  {e['name']}")
    for e in sorted(gpu, key=lambda e: e["ts"]):
        if r0 - 3000 <= e["ts"] < r1:
            nm = e["name"][:60]
            by = e.get("args", {}).get("bytes")
            bw = f" {by / e['dur'] / 1e3:6.1f} GB/s" if by and e["dur"] else ""
            print(f"   s{e.get('tid', '?'):<4} {(e['ts'] - r0) / 1e3:7.3f} +{e['dur'] / 1e3:6.3f}  {nm}{bw}")
