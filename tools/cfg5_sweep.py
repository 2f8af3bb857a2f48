"""BASELINE configs[4]: inter-device validation + apply sweep — CPU write logs of
1 MiB .. 4 GiB over a 64 GiB STMR sharded across G GPUs (not the bench line;
results go to profiles/).

One B200 per call in this environment, so each G is measured as ONE shard of
that configuration: 2^33/G words (64/G GiB; cells 4x that) holding the
entries routed to it — L/G of the global log, uniform over the shard.  Per
shard we time (CUDA events, library brackets): the router over the rank's
ingested 1/G (route_log_dptr, G buckets), validate+apply (apply_kernel +
restore_kernel), and validate-only (early validation).  The G-GPU aggregate
is G x the per-shard rate; the NCCL all-to-all of the buckets is NOT measured
here (it is estimated from the measured 770 GB/s NVLink peer copy, labelled).

    python tools/cfg5_sweep.py [--gs 2,4,8] [--logs-mib 1,4,16,64,256,1024,4096]
"""
import argparse
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_1905_00661_b200 as hetm

ENTRY = 24
ALG = 120  # algorithmic bytes per applied entry
NVLINK_GBS = 770.0  # measured peer copy per direction (B200_PROFILING.md), for the exchange estimate


def timed(dev, pre, fn, which, reps):
    ms = []
    for r in range(reps + 1):
        dev.clear_round()  # rolls the TS floor: every rep is a fresh round (no raced re-stores)
        pre(r)             # re-seed the RS bitmap, fresh ts (outside the timed launch)
        torch.cuda.synchronize()
        dev.set_timing(True)
        fn(r)
        dev.sync()
        t, c = dev.timing(which)
        dev.set_timing(False)
        if r:
            ms.append(t)
    return statistics.median(ms)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gs", default="2,4,8")
    ap.add_argument("--logs-mib", default="1,4,16,64,256,1024,4096")
    ap.add_argument("--reps", type=int, default=3)
    a = ap.parse_args()
    total_words = 1 << 33
    out = []
    for G in [int(x) for x in a.gs.split(",")]:
        W = total_words // G
        dev = hetm.GpuDevice(W, rs_gran_bytes=1024, shadow=False, log_capacity=1 << 20)
        # RS bitmap at density 1e-3 of its bits
        nbits = W * 8 // 1024
        rng = np.random.default_rng(G)
        bits = rng.integers(0, nbits, max(1, nbits // 1000)).astype(np.uint64)
        rs = np.zeros((nbits + 63) // 64, np.uint64)
        np.bitwise_or.at(rs, (bits >> np.uint64(6)).astype(np.int64), np.left_shift(np.uint64(1), bits & np.uint64(63)))
        dev.or_bitmap(hetm.BMP_RS, rs)
        g = torch.Generator(device="cuda").manual_seed(G)
        ts_next = 1
        for mib in [int(x) for x in a.logs_mib.split(",")]:
            n_global = (mib << 20) // ENTRY
            n = n_global // G  # entries this shard owns (uniform global log)
            log = torch.empty((n, 3), dtype=torch.int64, device="cuda")
            log[:, 0] = torch.randint(0, W, (n,), device="cuda", generator=g)
            log[:, 1] = torch.randint(-(1 << 62), 1 << 62, (n,), device="cuda", generator=g)
            routed = torch.empty_like(log)
            counts = torch.zeros(G, dtype=torch.int64, device="cuda")
            ingest = log.clone()  # the rank's 1/G of the global log, addresses over all shards
            ingest[:, 0] = torch.randint(0, total_words, (n,), device="cuda", generator=g)

            def fresh(r):
                nonlocal ts_next
                dev.or_bitmap(hetm.BMP_RS, rs)
                log[:, 2] = torch.arange(ts_next, ts_next + n, device="cuda")
                ts_next += n

            def apply(r):
                dev.validate_dptr(log.data_ptr(), n, hetm.APPLY)

            def vonly(r):
                dev.validate_dptr(log.data_ptr(), n, hetm.VALIDATE_ONLY)

            rstream = torch.cuda.Stream()

            def route(r):
                dev.route_log_dptr(ingest.data_ptr(), n, G, W, routed.data_ptr(), counts.data_ptr(),
                                   rstream.cuda_stream)

            ms_apply = timed(dev, fresh, apply, 1, a.reps)
            conflict = dev.round_verdict()
            ms_vonly = timed(dev, fresh, vonly, 1, a.reps)
            dev.clear_round()
            torch.cuda.synchronize()
            ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            rt = []
            for r in range(a.reps + 1):
                ev0.record(rstream)
                route(r)
                ev1.record(rstream)
                torch.cuda.synchronize()
                if r:
                    rt.append(ev0.elapsed_time(ev1))
            ms_route = statistics.median(rt)
            # fused route + delivery kernel with every owner's arena local (kernel cost;
            # across GPUs the stores go over NVLink, estimated below)
            ent, cnt = dev.recv_arena(G, n)
            pt = []
            for r in range(a.reps + 1):
                ev0.record(rstream)
                dev.route_to_peers_dptr(ingest.data_ptr(), n, G, W, 0, n, r & 1, [ent] * G, [cnt] * G,
                                        rstream.cuda_stream)
                ev1.record(rstream)
                torch.cuda.synchronize()
                if r:
                    pt.append(ev0.elapsed_time(ev1))
            ms_peer = statistics.median(pt)
            xchg_bytes = n * ENTRY * (G - 1) / G  # entries leaving this rank
            row = {
                "G": G, "shard_gib_words": W * 8 / 2**30, "log_mib_global": mib, "entries_per_shard": n,
                "apply_ms": ms_apply, "apply_gentries_s": n / ms_apply / 1e6,
                "apply_alg_gbs_per_gpu": ALG * n / ms_apply / 1e6,
                "apply_alg_gbs_aggregate": G * ALG * n / ms_apply / 1e6,
                "log_gbs_aggregate": G * ENTRY * n / ms_apply / 1e6,
                "validate_only_ms": ms_vonly, "validate_only_log_gbs_per_gpu": ENTRY * n / ms_vonly / 1e6,
                "route_ms": ms_route, "route_gbs_per_gpu": 2 * ENTRY * n / ms_route / 1e6,
                "route_to_peers_ms_local": ms_peer,
                "exchange_ms_estimate_nvlink": xchg_bytes / (NVLINK_GBS * 1e6),
                "conflict": bool(conflict),
            }
            out.append(row)
            print(json.dumps(row), flush=True)
            del log, routed, ingest
            torch.cuda.empty_cache()
        dev.close()
    return out


if __name__ == "__main__":
    main()
