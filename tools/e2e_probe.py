"""Phase timing of the bench's end-to-end round (not product code).

    python tools/e2e_probe.py [--chunk-merge]
"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import ctypes as C

import numpy as np

import paper_1905_00661_b200 as hetm

W, B, L = 1 << 27, 1 << 20, 1 << 20
delta = "--chunk-merge" not in sys.argv
dev = hetm.GpuDevice(W, rs_gran_bytes=1024, log_capacity=L, merge_delta=delta)
dev.register_kernel(hetm.KERNEL_BANK)
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
    hetm.gen_host_log(900 + j, L // 2, 2, 8, W // 2, W // 2, ts_base=1 + j * L, out=p.array)
tickets = hetm.PinnedArray((B,), np.uint64)
lib = hetm._lib.lib
acc = {}


def tick(name, t0):
    t1 = time.perf_counter()
    acc.setdefault(name, []).append((t1 - t0) * 1e3)
    return t1


for j in range(steps):
    t = time.perf_counter()
    st = hetm._lib.BatchStats()
    hetm.check(lib.hetm_dev_execute_batch(dev.h, hetm.KERNEL_BANK, txs[j % 2].array.ctypes.data, 24, B,
                                          tickets.array.ctypes.data, C.byref(st)), dev.h)
    t = tick("execute_batch", t)
    dev.merge_wait()
    t = tick("merge_wait(prev)", t)
    lg = logs[j].array
    o = np.argsort(lg["ts"], kind="stable")  # the host STM's own replica writes (not timed work of the device)
    host.array[lg["addr"][o]] = lg["value"][o]
    t = time.perf_counter()
    for c in range(8):
        dev.stream_chunk(lg[c * (L // 8):(c + 1) * (L // 8)], src_thread=c, seq=c)
    t = tick("stream_chunks", t)
    assert not dev.round_verdict()
    t = tick("verdict", t)
    ms = dev.merge_commit(host.array)
    t = tick("merge_commit", t)
    dev.clear_round()
    t = tick("clear_round", t)
dev.merge_wait()
print("delta" if delta else "chunk", {k: [round(x, 2) for x in v[1:]] for k, v in acc.items()})
print("bytes_d2h last merge", ms.bytes_d2h, "kernel_ms", st.kernel_ms)
ok = (dev.download(hetm.REPLICA_DEV) == host.array).all()
print("host replica == device replica:", ok)
