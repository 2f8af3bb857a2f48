#!/usr/bin/env python
"""bench.py — Speculative HeTM GPU-side path on B200 (BASELINE.json metric).

Workload (BASELINE.json configs[1], per GPU): 1 GiB STMR shard (2^27 words),
one 2^20-transaction bank batch per round (4 reads / 2 writes, uniform, on the
GPU half of the shard), and the round's host write log (2^20 entries of
<addr,value,ts>, uniform over the host halves of ALL shards) validated against
the GPU read-set bitmap (1 KiB granules) with the TS-guarded apply.

One step = one synchronization round of the device side:
    executeBatch (bank kernel) -> [G>1: route log by owner shard + NCCL
    all-to-all] -> validateChunk(apply) -> round clear.
`value` = committed GPU tx/s over all ranks, device-timed with CUDA events,
inputs resident in HBM (rotating per-step buffers; 1 GiB STMR >> L2).
`e2e` = the same rounds through the C-ABI host-buffer calls: H2D batch input,
H2D log stream, verdict, D2H tickets, mergeCommit D2H of dirty chunks.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "committed GPU tx/s (synthetic bank) 1 B200; validate+apply GB/s at 1/2/4/8 GPUs"
UNIT = "tx/s"
TX_BYTES = 224     # 24 B input + 8 B ticket + 4x32 B STMR sector reads + 2x32 B write-backs
ENTRY_BYTES = 120  # 24 B log + 32 B TS read + 32 B TS write + 32 B STMR sector write


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=20)
    p.add_argument("--warmup", type=int, default=5)
    p.add_argument("--impl", choices=["ours", "reference"], default="ours")
    p.add_argument("--words-log2", type=int, default=27)
    p.add_argument("--batch", type=int, default=1 << 20)
    p.add_argument("--log-entries", type=int, default=1 << 20)
    p.add_argument("--gran", type=int, default=1024)
    p.add_argument("--l2-fetch32", action="store_true", help="cudaLimitMaxL2FetchGranularity = 32 B")
    p.add_argument("--e2e-steps", type=int, default=20)
    p.add_argument("--no-early-merge", dest="early_merge", action="store_false",
                   help="e2e: merge only after the verdict (no hetm_dev_merge_prepare)")
    p.add_argument("--chunk-merge", action="store_true", help="SPEC chunk-copy merge instead of the delta merge")
    p.add_argument("--cpu-seconds", type=float, default=8.0)
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--no-preroll", action="store_true", help="skip the clock-sampling pre-roll (profiling runs)")
    return p.parse_args()


# ---------------------------------------------------------------- clocks
REASONS = ["gpu_idle", "applications_clocks_setting", "sw_power_cap", "hw_slowdown", "sync_boost",
           "sw_thermal_slowdown", "hw_thermal_slowdown", "hw_power_brake_slowdown"]


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled DURING the timed region."""

    def __init__(self, device: int):
        self.device = device
        self.proc = None
        self.lines = []

    def __enter__(self):
        q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.device), f"--query-gpu={q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except FileNotFoundError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *exc):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], 0, set()
        for ln in self.lines:
            parts = [x.strip() for x in ln.split(",")]
            try:
                sm.append(float(parts[0]))
                mx = max(mx, float(parts[1]))
                act = int(parts[2], 16)
            except (ValueError, IndexError):
                continue
            for i, name in enumerate(REASONS):
                if act & (1 << i) and name != "gpu_idle":
                    reasons.add(name)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0,
                    "raw": self.lines[:3]}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": mx, "reasons": sorted(reasons), "samples": len(sm)}


# Random 16-B accesses on a 1 GiB footprint, measured on B200 (tools/microbench.cu,
# profiles/r01_microbench_random_access.txt): L2-missing loads and read-modify-writes per second.
RANDOM_LOAD_PER_S, RANDOM_RMW_PER_S = 42.6e9, 22.6e9


def access_ceiling(tx_per_s, traffic, kernel_ms, peak):
    """The bank kernel's access-pattern bound beside the copy roofline: a transfer
    needs 4 random cell loads (P1) and 2 random RMWs of written cells (lock CAS,
    then the 128-bit commit store hitting the same line) — no schedule of the
    protocol issues fewer line fills.  Model time per tx = 4/load rate + 2/RMW rate."""
    ceil = 1.0 / (4 / RANDOM_LOAD_PER_S + 2 / RANDOM_RMW_PER_S)
    out = {"model": "4 random loads + 2 random RMWs per tx at the measured random-access rates",
           "load_per_s": RANDOM_LOAD_PER_S, "rmw_per_s": RANDOM_RMW_PER_S,
           "source": "profiles/r01_microbench_random_access.txt", "tx_per_s_ceiling": ceil,
           "kernel_tx_per_s": tx_per_s, "frac": tx_per_s / ceil}
    if traffic:
        dram_gbs = traffic / (kernel_ms * 1e-3) / 1e9
        out.update({"dram_gbs": dram_gbs, "dram_frac_of_peak": dram_gbs / peak})
    return out


NOMINAL_HBM_GBS = 8000.0  # north_star's nominal B200 HBM3e bandwidth (report both fractions)


def measured_traffic(kernel):
    """DRAM bytes per launch of `kernel` from the last committed ncu capture (profiles/traffic.json)."""
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as f:
            return json.load(f)[kernel]["bytes_per_launch"]
    except Exception:
        return None


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


# ----------------------------------------------------------- distributed
def dist_setup(args):
    """One process per GPU over NCCL.  HETM_BENCH_BACKEND=gloo with
    HETM_BENCH_ONE_GPU=1 runs the N-rank protocol with every rank on GPU 0
    (a functional test of the multi-rank path on a single-GPU box)."""
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if os.environ.get("HETM_BENCH_ONE_GPU") == "1":
        local = 0
    pg = None
    if world > 1:
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(local)
        backend = os.environ.get("HETM_BENCH_BACKEND", "nccl")
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
        pg = dist
    return world, rank, local, pg


def all_reduce(dist, t, op=None):
    """all_reduce that also works for a CPU-only backend (gloo test mode)."""
    import torch

    if os.environ.get("HETM_BENCH_BACKEND", "nccl") == "nccl":
        dist.all_reduce(t, op=op) if op is not None else dist.all_reduce(t)
        return t
    c = t.cpu()
    dist.all_reduce(c, op=op) if op is not None else dist.all_reduce(c)
    return c.to(t.device)


def host_log_slice(hetm, seed, n_entries, world, W, rank, ts_base):
    """This rank's 1/G of the global host log: uniform over the host halves
    [s*W + W/2, (s+1)*W) of every shard s; 2 writes per host tx."""
    n_tx = n_entries // 2
    log = hetm.gen_host_log(seed, n_tx, 2, 8, 0, world * (W // 2), ts_base=ts_base)
    v = log["addr"]
    shard = v // np.uint64(W // 2)
    log["addr"] = shard * np.uint64(W) + np.uint64(W // 2) + (v % np.uint64(W // 2))
    return log


# -------------------------------------------------------------- our arm
def run_ours(args):
    import torch

    import paper_1905_00661_b200 as hetm
    from paper_1905_00661_b200.shard import PeerValidator, ShardedValidator

    world, rank, local, dist = dist_setup(args)
    torch.cuda.set_device(local)
    W = 1 << args.words_log2
    base = rank * W
    B, L = args.batch, args.log_entries
    K, WU = args.steps, args.warmup
    n_steps = K + WU

    dev = hetm.GpuDevice(W, shard_base=base, rs_gran_bytes=args.gran, device=local, log_capacity=max(L, 1 << 20),
                         l2_fetch_32=args.l2_fetch32, merge_delta=not args.chunk_merge)
    dev.register_kernel(hetm.KERNEL_BANK)
    init = np.full(W, 1000, np.uint64)
    dev.upload(hetm.REPLICA_DEV, base, init)
    host_replica = hetm.PinnedArray((W,), np.uint64)
    host_replica.array[:] = init
    dev.merge_commit(host_replica.array)  # shadow == round start, host replica aligned
    dev.merge_wait()
    dev.clear_round()

    # ---- rotating per-step inputs, resident in HBM (total > L2)
    t_gen = time.time()
    n_bufs = min(n_steps, 16)
    tx_d, log_d = [], []
    for j in range(n_bufs):
        txs = hetm.gen_bank_batch(1000 + 7919 * rank + j, B, base, W // 2)
        tx_d.append(torch.from_numpy(txs.view(np.uint8)).cuda())
    base_log = host_log_slice(hetm, 77 + rank, L, world, W, rank, ts_base=0)
    base_log_t = torch.from_numpy(base_log.view(np.uint64).reshape(-1, 3).astype(np.int64)).cuda()
    for j in range(n_steps):
        t = base_log_t.clone()
        t[:, 2] += (j * world + rank) * (L // 2) + 1  # unique, monotone ts across ranks and steps
        log_d.append(t)
    tickets = torch.empty(B, dtype=torch.int64, device="cuda")
    gen_s = time.time() - t_gen

    s_exec = dev.stream_handle(0)
    s_val = dev.stream_handle(2)
    ex = torch.cuda.ExternalStream(s_exec)
    vs = torch.cuda.ExternalStream(s_val)
    exchange = "none (1 shard)"
    sv = None
    if world > 1:  # fused router + NVLink delivery into the owners' arenas; NCCL all_to_all as the fallback
        try:
            sv = PeerValidator(dev, world, rank, W, L, dist, s_val)
            exchange = "fused router -> NVLink peer stores (CUDA IPC arenas)"
        except RuntimeError:
            sv = None
    if sv is None:
        sv = ShardedValidator(dev, world, W, L, dist, s_val)
        if world > 1:
            exchange = "router -> NCCL all_to_all"


    def step(j, timed_idx=None):
        tb = tx_d[j % n_bufs]
        dev.execute_batch_dptr(hetm.KERNEL_BANK, tb.data_ptr(), B, tickets.data_ptr(), s_exec)
        lg = log_d[j]
        with torch.cuda.stream(vs):  # router, exchange and validation share the validation stream
            n_local = sv.validate(lg, hetm.APPLY)
        if n_local is None:  # fused peer exchange on NCCL: counts stay on the device; every entry has one owner
            n_local = L
        dev.clear_round(asynchronous=True)
        return n_local

    for j in range(WU):
        step(j)
    conflict, _ = dev.read_counters()
    assert not conflict, "partitioned bank workload must not conflict"
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    start, stop = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    n_val = 0
    with ClockSampler(local) as clk:
        # pre-roll under the same load so nvidia-smi has samples spanning the timed region
        t_pre = time.time()
        j = 0
        while not args.no_preroll and time.time() - t_pre < 0.6:
            step(j % WU if WU else 0)
            j += 1
            if j % 8 == 0:
                torch.cuda.synchronize()
        torch.cuda.synchronize()
        dev.timing(0), dev.timing(1)
        dev.set_timing(True)  # CUDA-event brackets around every batch / validation launch
        start.record(ex)
        for i in range(K):
            n_val += step(WU + i, i)
        # join every device stream back into s_exec before the stop event
        for sidx in (1, 2, 3, 4):
            other = torch.cuda.ExternalStream(dev.stream_handle(sidx))
            e = torch.cuda.Event()
            e.record(other)
            ex.wait_event(e)
        stop.record(ex)
        torch.cuda.synchronize()
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    ms_total = start.elapsed_time(stop)
    conflict, st = dev.read_counters()
    assert not conflict
    bt, bc = dev.timing(0)
    vt, vc = dev.timing(1)
    dev.set_timing(False)
    batch_ms, val_ms = bt / max(bc, 1), vt / K  # validation: all launches of a step (G regions with the peer exchange)
    if dist:
        t = torch.tensor([ms_total, batch_ms, val_ms], dtype=torch.float64, device="cuda")
        t = all_reduce(dist, t, op=dist.ReduceOp.MAX)
        ms_total, batch_ms, val_ms = t.tolist()
        nv = torch.tensor([n_val], dtype=torch.int64, device="cuda")
        nv = all_reduce(dist, nv)
        n_val = int(nv.item())

    # correctness spot check after timing: bank sum preserved on the device
    dev_words = dev.download(hetm.REPLICA_DEV, base + 0, W // 2)
    bank_sum_ok = int(dev_words.sum(dtype=np.uint64)) == 1000 * (W // 2)

    # ---- end-to-end through the host-buffer C-ABI (pinned host memory)
    e2e = run_e2e(args, hetm, dev, host_replica, world, rank, W, base, dist)

    ms_step = ms_total / K
    # our kernels per step (the ncu launch list in profiles/ shows the same set):
    # bank_batch_kernel (+ the AUTO schedule's side-stream hot_estimate_kernel), apply_kernel +
    # restore_kernel, clear_round_kernel (async clear: bitmaps zeroed + round counters rolled)
    launches_detail = {"bank_batch_kernel": 1, "hot_estimate_kernel": 1, "apply_kernel": 1, "restore_kernel": 1,
                       "clear_round_kernel": 1}
    if world > 1 and isinstance(sv, PeerValidator):
        launches_detail.update({"route_count_kernel": 1, "route_scan_kernel": 1, "route_peer_publish_kernel": 1,
                                "route_peer_scatter_kernel": 1})
    elif world > 1:
        launches_detail.update({"route_count_kernel": 1, "route_scan_kernel": 1, "route_scatter_kernel": 1})
    launches_per_step = sum(launches_detail.values())
    value = world * B * K / (ms_total / 1e3)
    peak, peak_kind = peaks()
    achieved = TX_BYTES * B / (batch_ms * 1e-3) / 1e9
    val_gbs = ENTRY_BYTES * (n_val / K / world) / (val_ms * 1e-3) / 1e9
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": K, "warmup": WU,
        "ms_per_step": ms_step, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "u64", "data": "synthetic (seeded DetRng bank batches + host write logs)",
        "config": {
            "workload": "BASELINE configs[1]: bank, 1 GiB STMR per GPU, 2^20-tx GPU batch per round, 4R/2W "
                        "uniform, RS/WS gran 1 KiB; round host log 2^20 entries on the host halves, "
                        "validated+applied (routed by owner shard over NCCL when G>1)",
            "stmr_words_per_gpu": W, "batch_tx": B, "log_entries_per_gpu": L, "rs_gran_bytes": args.gran,
            "stmr_layout": "16-B word cells {value, lock-or-TS}", "parallelism": f"shard{world}",
            "log_exchange": exchange,
            "l2": "inputs larger than L2: 1 GiB STMR per GPU, rotating per-step input buffers "
                  f"({n_bufs} tx batches + {n_steps} logs, {(n_bufs * B * 24 + n_steps * L * 24) >> 20} MiB)",
        },
        "roofline": {"bound": "hbm", "kernel": "bank_batch_kernel", "achieved": achieved, "peak": peak,
                     "peak_kind": peak_kind, "unit": "GB/s", "frac": achieved / peak,
                     "peak_nominal": NOMINAL_HBM_GBS, "frac_nominal": achieved / NOMINAL_HBM_GBS,
                     "traffic": measured_traffic("bank_batch_kernel"),
                     "traffic_source": "profiles/traffic.json (ncu --set full, dram read+write per launch)",
                     "algorithmic_bytes_per_tx": TX_BYTES, "kernel_ms": batch_ms,
                     "access_pattern_ceiling": access_ceiling(B / (batch_ms * 1e-3), measured_traffic("bank_batch_kernel"),
                                                              batch_ms, peak)},
        "validate_apply": {"kernel": "apply_kernel", "gbs_algorithmic": val_gbs,
                           "entries_per_s_per_gpu": (n_val / K / world) / (val_ms / 1e3),
                           "log_gbs_per_gpu": 24 * (n_val / K / world) / (val_ms * 1e-3) / 1e9,
                           "frac": val_gbs / peak, "frac_nominal": val_gbs / NOMINAL_HBM_GBS,
                           "algorithmic_bytes_per_entry": ENTRY_BYTES,
                           "traffic": measured_traffic("validate_apply"),
                           "kernel_ms": val_ms, "aggregate_gbs": val_gbs * world},
        "batch": {"committed_last": int(st.committed), "aborts_last": int(st.aborts)},
        "bank_sum_ok": bank_sum_ok,
        "e2e": e2e,
        "gpu_launches": K * launches_per_step,
        "gpu_launches_per_step": launches_detail,
        "clocks": clk.summary(),
        "input_gen_s": gen_s,
    }
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(args, seconds=args.cpu_seconds)
    if rank == 0:
        print(json.dumps(line), flush=True)
    dev.close()
    if dist:
        dist.barrier()
        dist.destroy_process_group()


def run_e2e(args, hetm, dev, host_replica, world, rank, W, base, dist):
    """Full synchronous rounds through the public C-ABI with HOST buffers."""
    B, L = args.batch, args.log_entries
    steps = args.e2e_steps
    txs = [hetm.PinnedArray((B,), hetm.BANK_TX) for _ in range(2)]
    for j, p in enumerate(txs):
        hetm.gen_bank_batch(555 + j + 31 * rank, B, base, W // 2, out=p.array)
    logs = [hetm.PinnedArray((L,), hetm.LOG_ENTRY) for _ in range(steps + 1)]
    ts0 = 10_000_000_000
    for j, p in enumerate(logs):  # produced by host txs before the round: not timed
        hetm.gen_host_log(900 + j, L // 2, 2, 8, base + W // 2, W // 2, ts_base=ts0 + j * L, out=p.array)
    info = dev.info()
    dev.sync()
    conflict, _ = dev.read_counters()
    dev.clear_round()  # synchronous clear: refresh the TS floor after the pipelined rounds
    tickets = hetm.PinnedArray((B,), np.uint64)
    import ctypes as C
    lib = hetm._lib.lib
    h2d = d2h = 0
    if dist:
        dist.barrier()
    t0 = time.perf_counter()
    for j in range(steps + 1):
        if j == 1:  # first round is warm-up
            dev.merge_wait()
            if dist:
                dist.barrier()
            t0 = time.perf_counter()
            h2d = d2h = 0
        lg = logs[j].array
        st = hetm._lib.BatchStats()
        # the GPU resumes right away: this batch overlaps the
        # previous round's merge landing in the host replica
        rc = lib.hetm_dev_execute_batch(dev.h, hetm.KERNEL_BANK, txs[j % 2].array.ctypes.data, 24, B,
                                        tickets.array.ctypes.data, C.byref(st))
        hetm.check(rc, dev.h)
        # execution phase over: stage this round's delta merge now and apply it to
        # the host replica speculatively (undone on abort); this waits for the
        # previous round's merge to have landed, so host transactions of this
        # round saw the merged replica
        if args.early_merge:
            dev.merge_prepare(host_replica.array)
        else:
            dev.merge_wait()
        for c in range(8):  # the round's log streamed in 8 chunks (one per host thread)
            sl = lg[c * (L // 8):(c + 1) * (L // 8)]
            dev.stream_chunk(sl, src_thread=c, seq=c)
        conflict = dev.round_verdict()
        if conflict:
            raise RuntimeError("unexpected conflict in the partitioned e2e round")
        ms = dev.merge_commit(host_replica.array)
        dev.clear_round()
        h2d += B * 24 + L * 24
        d2h += B * 8 + ms.bytes_d2h
    dev.merge_wait()
    dt = time.perf_counter() - t0
    if dist:
        import torch
        t = torch.tensor([dt], dtype=torch.float64, device="cuda")
        t = all_reduce(dist, t, op=dist.ReduceOp.MAX)
        dt = float(t.item())
    for p in txs + logs + [tickets]:
        p.free()
    return {"value": world * B * steps / dt, "unit": UNIT, "h2d_bytes_per_step": h2d // steps,
            "d2h_bytes_per_step": d2h // steps, "steps": steps, "ms_per_step": dt / steps * 1e3,
            "merge": ("chunk copy (SPEC.md:363-371)" if args.chunk_merge else
                      "delta (12-B {word,value} per device-written word)" +
                      (", staged + speculatively applied right after the execution phase (hetm_dev_merge_prepare)"
                       if args.early_merge else "")),
            "bound": "host DRAM: the merge scatter of ~2^21 random words into the host replica per round plus "
                     "the DMAs (profiles/r01_e2e_bounds.txt)",
            "timing": "host wall clock around full rounds (pinned buffers; verdict + merge D2H landed in the host "
                      "replica before the next round's host log; the next GPU batch overlaps the merge, PAPER.md:355)"}


# ---------------------------------------------------------- CPU baseline
def cpu_baseline(args, seconds=8.0, rounds=None):
    """The reference CPU path (oracle port, multi-threaded) on a bounded sample
    of the same round: one bank batch (guest-stm-batch worker pool)
    + validate/apply of the round's log on all host threads."""
    import oracle as O

    threads = os.cpu_count() or 1
    W = 1 << args.words_log2
    B = args.batch // 4
    L = args.log_entries // 4
    s = np.full(W, 1000, np.uint64)
    ts = np.zeros(W, np.uint64)
    gran = args.gran
    rs = np.zeros(((W * 8 // gran) + 63) // 64, np.uint64)
    done_tx, t_tot, r = 0, 0.0, 0
    while (rounds is None and t_tot < seconds) or (rounds is not None and r < rounds):
        txs = O.gen_bank_batch(3000 + r, B, 0, W // 2)
        log = O.gen_host_log(4000 + r, L // 2, 2, 8, W // 2, W // 2, ts_base=r * L)
        rs[:] = 0
        t0 = time.perf_counter()
        c, _, rsb, _, _ = O.mt_bank_batch(s, txs, threads, lock_entries=1 << 24, gran=gran, tickets=False)
        O.mt_validate_apply(log, rsb, gran, ts, s, threads)
        t_tot += time.perf_counter() - t0
        done_tx += c
        r += 1
    return {"value": done_tx / t_tot, "unit": UNIT, "cores": threads, "kind": "port",
            "sample": f"{r} rounds x ({B} bank tx + {L} log entries) on the 2^{args.words_log2}-word STMR "
                      f"(1/4 of a GPU round), oracle/hetm_oracle.c pthreads",
            "host": host_info()}


def host_info():
    """the CPU the baseline ran on (hardware_concurrency, model, MemTotal)."""
    info = {"nproc": os.cpu_count()}
    try:
        info["affinity_cpus"] = len(os.sched_getaffinity(0))
    except Exception:
        pass
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                info["cpu_model"] = line.split(":", 1)[1].strip()
                break
        for line in open("/proc/meminfo"):
            if line.startswith("MemTotal"):
                info["mem_total_gb"] = round(int(line.split()[1]) / (1 << 20), 1)
                break
    except OSError:
        pass
    return info


def run_reference(args):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    # warmup rounds untimed, then K timed rounds
    import oracle  # noqa: F401  (builds the checker if needed)
    cpu_baseline(args, rounds=max(1, args.warmup // 2))
    t0 = time.perf_counter()
    cb = cpu_baseline(args, rounds=args.steps)
    dt = time.perf_counter() - t0
    line = {"metric": METRIC, "value": cb["value"], "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": dt / args.steps * 1e3, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "u64", "data": "synthetic",
            "impl": "reference",
            "config": {"workload": "BASELINE configs[1] (bounded per-step sample, see cpu_baseline.sample)",
                       "stmr_words": 1 << args.words_log2},
            "cpu_baseline": cb,
            "e2e": {"value": cb["value"], "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
