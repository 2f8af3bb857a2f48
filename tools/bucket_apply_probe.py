"""Probe: does grouping a host write log by address range before the apply
pass help validate+apply on big shards?  (TLB reach: random 16-B cells over
128 GiB of cells run at ~5 G entries/s vs ~15 G/s over 64 GiB.)

For each shard size and log size: apply of the raw uniform log vs route into B
contiguous address buckets (hetm_dev_route_log_dptr, the shard router run on
one shard's sub-ranges) + apply of the routed log.  CUDA events on the
validation stream, median of reps.  Usage:
  python tools/bucket_apply_probe.py [words_log2 ...]
"""
import statistics
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_1905_00661_b200 as hetm  # noqa: E402


def run(words_log2, log_entries, buckets_list, reps=3):
    W = 1 << words_log2
    d = hetm.GpuDevice(W, rs_gran_bytes=1024, shadow=False, log_capacity=1 << 20)
    s_val = d.stream_handle(2)
    vs = torch.cuda.ExternalStream(s_val)
    g = torch.Generator(device="cuda").manual_seed(7)
    n = log_entries
    log = torch.empty((n, 3), dtype=torch.int64, device="cuda")
    log[:, 0] = torch.randint(0, W, (n,), device="cuda", generator=g)
    log[:, 1] = torch.randint(-(1 << 62), 1 << 62, (n,), device="cuda", generator=g)
    routed = torch.empty_like(log)
    counts = torch.zeros(64, dtype=torch.int64, device="cuda")
    ts = [1]
    ev0, ev1, evm = (torch.cuda.Event(enable_timing=True) for _ in range(3))

    def fresh_ts():
        d.clear_round()
        log[:, 2] = torch.arange(ts[0], ts[0] + n, device="cuda", dtype=torch.int64)
        ts[0] += n
        torch.cuda.synchronize()

    out = []
    for B in [1] + buckets_list:
        t_all, t_route = [], []
        for r in range(reps + 1):
            fresh_ts()
            ev0.record(vs)
            if B == 1:
                d.validate_dptr(log.data_ptr(), n, hetm.APPLY, s_val)
                evm.record(vs)
            else:
                d.route_log_dptr(log.data_ptr(), n, B, W // B, routed.data_ptr(), counts.data_ptr(), s_val)
                evm.record(vs)
                d.validate_dptr(routed.data_ptr(), n, hetm.APPLY, s_val)
            ev1.record(vs)
            torch.cuda.synchronize()
            if r:
                t_all.append(ev0.elapsed_time(ev1))
                t_route.append(ev0.elapsed_time(evm))
        ms = statistics.median(t_all)
        rms = statistics.median(t_route) if B > 1 else 0.0
        line = (f"W=2^{words_log2} ({(W * 16) >> 30} GiB cells) n={n:>10} B={B:>3}: total {ms:8.3f} ms "
                f"(route {rms:6.3f})  {n / ms / 1e6:6.2f} G entries/s")
        print(line, flush=True)
        out.append(line)
    d.close()
    del log, routed
    torch.cuda.empty_cache()
    return out


if __name__ == "__main__":
    sizes = [int(a) for a in sys.argv[1:]] or [27, 31, 32, 33]
    for wl in sizes:
        for n in (1 << 20, 44739242):
            if n > (1 << wl):
                continue
            run(wl, n, [4, 16, 64])
