"""Kernel probes for tuning (not product code).  HETM_KNOCKOUT variants need the experiments
build: make -C paper_1905_00661_b200/csrc clean all EXPERIMENTS=1.

    python tools/probe_r02.py bank            # bank batch kernel ms (HETM_KNOCKOUT selects variants)
    python tools/probe_r02.py val [log2 n]    # validate+apply ms per chunk (HETM_VAL_WINDOW_LOG2)
"""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_1905_00661_b200 as hetm

W = 1 << int(os.environ.get("PROBE_WORDS_LOG2", "27"))


def bank():
    B = 1 << 20
    d = hetm.GpuDevice(W, rs_gran_bytes=1024)
    d.register_kernel(hetm.KERNEL_BANK)
    d.upload(hetm.REPLICA_DEV, 0, np.full(W, 1000, np.uint64))
    ms, ab = [], []
    tk = torch.empty(B, dtype=torch.int64, device="cuda")
    for rep in range(6):  # device-resident inputs: one 2^20-tx launch, as in bench.py's timed loop
        txs = torch.from_numpy(hetm.gen_bank_batch(10 + rep, B, 0, W // 2).view(np.uint8)).cuda()
        d.set_timing(True)
        d.execute_batch_dptr(hetm.KERNEL_BANK, txs.data_ptr(), B, tk.data_ptr())
        d.sync()
        t, _ = d.timing(0)
        d.set_timing(False)
        _, st = d.read_counters()
        d.clear_round()
        if rep:
            ms.append(t)
            ab.append(st.aborts)
    out = np.zeros(6, np.uint64)
    hetm.check(hetm._lib.lib.hetm_dev_debug_words(d.h, out.ctypes.data, 6))
    ko = os.environ.get("HETM_KNOCKOUT", "0")
    print(f"bank KO={ko} kernel_ms median {statistics.median(ms):.4f} min {min(ms):.4f} "
          f"aborts {statistics.median(ab):.0f} tx/s {B / statistics.median(ms) / 1e6:.2f} G "
          f"ticket_atomics(total,6 batches) {int(out[4])}")


def val(log2n):
    n = 1 << log2n
    d = hetm.GpuDevice(W, rs_gran_bytes=1024, log_capacity=n)
    log = hetm.gen_host_log(5, n // 2, 2, 8, 0, W, ts_base=0)
    base = torch.from_numpy(log.view(np.uint64).reshape(-1, 3).astype(np.int64)).cuda()
    ms = []
    for rep in range(8):
        t = base.clone()
        t[:, 2] += rep * n + 1
        torch.cuda.synchronize()
        d.set_timing(True)
        d.validate_dptr(t.data_ptr(), n, hetm.APPLY)
        d.sync()
        tm, c = d.timing(1)
        d.set_timing(False)
        d.clear_round()
        if rep:
            ms.append(tm)
    # spot check: the last chunk's values are in place where its ts is the max
    got = d.download(hetm.REPLICA_DEV, 0, W)
    last = t.cpu().numpy().view(np.uint64)
    okv = (got[last[:, 0].astype(np.int64)] == last[:, 1]).mean()
    med = statistics.median(ms)
    wl = os.environ.get("HETM_VAL_WINDOW_LOG2", "18")
    print(f"val n=2^{log2n} window=2^{wl} ms median {med:.4f} min {min(ms):.4f} "
          f"{n / med / 1e6:.2f} G entries/s {120 * n / med / 1e6:.0f} GB/s alg; last-chunk values ok {okv:.4f}")


if __name__ == "__main__":
    if sys.argv[1] == "bank":
        bank()
    else:
        val(int(sys.argv[2]) if len(sys.argv) > 2 else 20)
