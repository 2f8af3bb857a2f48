#!/usr/bin/env python
"""bench.py — Speculative HeTM GPU-side path on B200 (BASELINE.json metric:
"committed GPU tx/s (synthetic bank) 1 B200; validate+apply GB/s at 1/2/4/8 GPUs").

Headline workload (BASELINE.json configs[1], per GPU): 1 GiB STMR shard (2^27
words), one 2^20-transaction bank batch per round (4 reads / 2 writes,
uniform, on the GPU half of the shard), and the round's host write log (2^20
entries of <addr,value,ts>, uniform over the host halves of ALL shards)
validated against the GPU read-set bitmap (1 KiB granules) with the
TS-guarded apply.

One step = one synchronization round of the device side:
    executeBatch (bank kernel) -> [G>1: fused route to the owner shards over
    NVLink] -> validateChunk(apply) -> device half of mergeCommit
    (hetm_dev_merge_stage: write-set records + devShadow refresh) -> round clear.
`value` = committed GPU tx/s over all ranks, device-timed with CUDA events,
inputs resident in HBM (rotating per-step buffers; 1 GiB STMR >> L2).
`e2e` = the same rounds through the C-ABI host-buffer calls: H2D batch input,
H2D log stream, verdict, D2H tickets, mergeCommit D2H into the host replica.
`e2e_live` = Engine::runRound with a LIVE TL2 host producer (build/hetm_live_round).
`configs` = BASELINE configs[2] (zipf 0.99, conflict + rollback rounds) and
configs[3] (cache GET/SET 90/10), device-resident, at N = 1.
`validate_apply` = BASELINE configs[4]: a 64 GiB STMR sharded 64/G GiB per GPU,
global CPU write logs of 16 MiB .. 4 GiB, each rank ingesting 1/G and routing
entries to their owner shard over NVLink (fused route kernel, peer stores),
then validate + TS-guarded apply; aggregate GB/s at every N.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

--gpus N > 1 without a torchrun environment re-launches itself under
`torch.distributed.run` with N ranks (one per GPU); fewer visible GPUs than N
is an error.  --plan prints the configuration line without touching a GPU.
"""
from __future__ import annotations

import argparse
import json
import os
import socket
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
LOG_ENTRY_WIRE = 24  # write_log.hpp:25 kLogEntryWireBytes
NOMINAL_HBM_GBS = 8000.0  # north_star's nominal B200 HBM3e bandwidth (report both fractions)


def one_gpu_mode() -> bool:
    return os.environ.get("HETM_BENCH_ONE_GPU") == "1"


def parse(argv=None):
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=20)
    p.add_argument("--warmup", type=int, default=5)
    p.add_argument("--impl", choices=["ours", "reference"], default="ours")
    p.add_argument("--plan", action="store_true", help="print the configuration line only (no GPU work)")
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
    p.add_argument("--live-rounds", type=int, default=12, help="e2e_live rounds (0: skip)")
    p.add_argument("--no-configs", action="store_true", help="skip the configs[2]/[3] sub-lines")
    p.add_argument("--config-rounds", type=int, default=8)
    p.add_argument("--cfg5-words-log2", type=int, default=None,
                   help="global STMR of the validate_apply sweep (default 2^33 = 64 GiB; 2^28 in one-GPU mode)")
    p.add_argument("--cfg5-log-mib", default=None,
                   help="global log sizes of the sweep, MiB (default 16,256,1024,4096; 1,16 in one-GPU mode)")
    p.add_argument("--cfg5-reps", type=int, default=3)
    p.add_argument("--no-cfg5", action="store_true")
    a = p.parse_args(argv)
    if a.cfg5_words_log2 is None:
        a.cfg5_words_log2 = 28 if one_gpu_mode() else 33
    if a.cfg5_log_mib is None:
        a.cfg5_log_mib = "1,16" if one_gpu_mode() else "16,256,1024,4096"
    return a


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


# ------------------------------------------------------------- rooflines
# Access floor of the stripe-lock bank kernel: the same 2^20 random transfers
# doing only what no protocol can avoid — load the two written 16-B cells and
# store them back (the read-only accounts' values are unused, their locks live
# in the L2-resident stripe table) — tools/stripe_probe.cu "floor" on B200,
# 1 CTA/SM: profiles/r02l_stripe_probe.txt.  The protocol (stripe locks,
# ticket, read-set validation, release fence, bitmaps) costs the difference.
PROTOCOL_FLOOR_MS = 0.1189


def protocol_floor(kernel_ms, traffic, peak):
    out = {"model": "same transfers, no protocol: 128-bit load + store of the two written cells only",
           "source": "profiles/r02l_stripe_probe.txt (tools/stripe_probe.cu floor)", "floor_kernel_ms": PROTOCOL_FLOOR_MS,
           "floor_tx_per_s": (1 << 20) / (PROTOCOL_FLOOR_MS * 1e-3),
           "kernel_over_floor": kernel_ms / PROTOCOL_FLOOR_MS}
    if traffic:
        dram_gbs = traffic / (kernel_ms * 1e-3) / 1e9
        out.update({"dram_gbs": dram_gbs, "dram_frac_of_peak": dram_gbs / peak})
    return out


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
def free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def maybe_spawn(args):
    """--gpus N honoured: outside torchrun, N > 1 re-launches this script under
    torch.distributed.run with N local ranks; inside it, WORLD_SIZE must be N."""
    env_world = os.environ.get("WORLD_SIZE")
    if env_world is not None:
        if int(env_world) != args.gpus and not (args.gpus == 1 and "--gpus" not in sys.argv):
            raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={env_world}")
        return
    if args.gpus <= 1:
        return
    if not args.plan and not one_gpu_mode() and args.impl == "ours":
        import torch
        have = torch.cuda.device_count()
        if have < args.gpus:
            raise SystemExit(f"bench.py: --gpus {args.gpus} needs {args.gpus} CUDA devices, {have} visible")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(free_port()), os.path.abspath(__file__),
           *sys.argv[1:]]
    sys.stdout.flush()
    os.execv(sys.executable, cmd)


def dist_setup():
    """One process per GPU over NCCL.  HETM_BENCH_BACKEND=gloo with
    HETM_BENCH_ONE_GPU=1 runs the N-rank protocol with every rank on GPU 0
    (a functional test of the multi-rank path on a single-GPU box)."""
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if one_gpu_mode():
        local = 0
    pg = None
    if world > 1:
        import torch
        import torch.distributed as dist
        backend = os.environ.get("HETM_BENCH_BACKEND", "nccl")
        if backend == "nccl":
            torch.cuda.set_device(local)
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
        pg = dist
    return world, rank, local, pg


def all_reduce(dist, t, op=None):
    """all_reduce that also works for a CPU-only backend (gloo test mode)."""
    if os.environ.get("HETM_BENCH_BACKEND", "nccl") == "nccl":
        dist.all_reduce(t, op=op) if op is not None else dist.all_reduce(t)
        return t
    c = t.cpu()
    dist.all_reduce(c, op=op) if op is not None else dist.all_reduce(c)
    return c.to(t.device)


def max_over_ranks(dist, values):
    """Element-wise max of a list of floats over all ranks (CPU tensors work for both backends)."""
    if not dist:
        return list(values)
    import torch
    if os.environ.get("HETM_BENCH_BACKEND", "nccl") == "nccl":
        t = torch.tensor(list(values), dtype=torch.float64, device="cuda")
    else:
        t = torch.tensor(list(values), dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return t.cpu().tolist()


def host_log_slice(hetm, seed, n_entries, world, W, rank, ts_base):
    """This rank's 1/G of the global host log: uniform over the host halves
    [s*W + W/2, (s+1)*W) of every shard s; 2 writes per host tx."""
    n_tx = n_entries // 2
    log = hetm.gen_host_log(seed, n_tx, 2, 8, 0, world * (W // 2), ts_base=ts_base)
    v = log["addr"]
    shard = v // np.uint64(W // 2)
    log["addr"] = shard * np.uint64(W) + np.uint64(W // 2) + (v % np.uint64(W // 2))
    return log


def cfg5_plan(args, world):
    """Geometry of the configs[4] sweep and the NVLink bytes it moves per round
    (DESIGN.md §6): each rank ingests 1/G of the global log; (G-1)/G of its
    entries belong to another shard and are stored into the owner's arena."""
    total = 1 << args.cfg5_words_log2
    out = []
    for mib in [int(x) for x in args.cfg5_log_mib.split(",")]:
        n_global = (mib << 20) // LOG_ENTRY_WIRE
        n_local = n_global // world
        out.append({"log_mib_global": mib, "entries_global": n_local * world, "entries_ingested_per_rank": n_local,
                    "nvlink_bytes_out_per_rank": int(n_local * LOG_ENTRY_WIRE * (world - 1) / world),
                    "nvlink_bytes_total": int(n_local * LOG_ENTRY_WIRE * (world - 1))})
    return {"stmr_words_global": total, "stmr_gib_global": total * 8 / 2**30, "shard_words": total // world,
            "shard_gib": total * 8 / 2**30 / world, "sizes": out}


# -------------------------------------------------------------- our arm
def run_ours(args):
    import torch

    import paper_1905_00661_b200 as hetm
    from paper_1905_00661_b200.shard import PeerValidator, ShardedValidator

    world, rank, local, dist = dist_setup()
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
    # entries validated from device memory join the round arena (HETM_RETAIN), so
    # the device half of mergeCommit refreshes devShadow incrementally
    val_mode = hetm.APPLY | (hetm.RETAIN if world == 1 else 0)
    merge_dev = not args.chunk_merge

    def step(j):
        tb = tx_d[j % n_bufs]
        dev.execute_batch_dptr(hetm.KERNEL_BANK, tb.data_ptr(), B, tickets.data_ptr(), s_exec)
        lg = log_d[j]
        with torch.cuda.stream(vs):  # router, exchange and validation share the validation stream
            n_local = sv.validate(lg, val_mode)
        if n_local is None:  # fused peer exchange on NCCL: counts stay on the device; every entry has one owner
            n_local = L
        if merge_dev:
            dev.merge_stage()  # device half of mergeCommit: write-set records + devShadow refresh
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
        # steps carry collectives at N>1 (verdict / delivery barrier), so every
        # rank must run the same number: the stop decision is taken every 8
        # steps and agreed over the ranks (a per-rank clock once left one rank
        # in a step's collective while the other waited in the barrier below)
        while not args.no_preroll:
            for _ in range(8):
                step(j % WU if WU else 0)
                j += 1
            torch.cuda.synchronize()
            done = 1.0 if time.time() - t_pre >= 0.6 else 0.0
            if dist:
                done = max_over_ranks(dist, [done])[0]
            if done > 0:
                break
        torch.cuda.synchronize()
        for w in (0, 1, 2):
            dev.timing(w)
        dev.set_timing(True)  # CUDA-event brackets around every batch / validation / merge-stage launch
        start.record(ex)
        for i in range(K):
            n_val += step(WU + i)
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
    mt, mc = dev.timing(2)
    dev.set_timing(False)
    batch_ms, val_ms, mstage_ms = bt / max(bc, 1), vt / K, mt / K
    if dist:
        ms_total, batch_ms, val_ms, mstage_ms = max_over_ranks(dist, [ms_total, batch_ms, val_ms, mstage_ms])
        nv = torch.tensor([n_val], dtype=torch.int64, device="cuda")
        nv = all_reduce(dist, nv)
        n_val = int(nv.item())

    # correctness spot checks after timing: bank sum preserved; devShadow == devReplica
    dev_words = dev.download(hetm.REPLICA_DEV, base + 0, W // 2)
    bank_sum_ok = int(dev_words.sum(dtype=np.uint64)) == 1000 * (W // 2)
    shadow_ok = None
    if merge_dev and world == 1:
        shadow_ok = bool((dev.download(hetm.REPLICA_DEV_SHADOW) == dev.download(hetm.REPLICA_DEV)).all())
    del tx_d, log_d, base_log_t
    torch.cuda.empty_cache()

    # ---- end-to-end through the host-buffer C-ABI (pinned host memory)
    e2e = run_e2e(args, hetm, dev, host_replica, world, rank, W, base, dist)
    ms_step = ms_total / K
    # our kernels per step (the ncu launch list in profiles/ shows the same set)
    launches_detail = {"bank_batch_kernel": 1, "hot_estimate_kernel": 1, "apply_xchg_kernel": 1}
    if merge_dev:
        # bank rounds carry per-word commit versions: the versioned pick pass (no claim bitmap)
        launches_detail.update({"delta_pick_kernel": 1, "delta_emit_kernel": 1, "winner_kernel": 1})
    launches_detail["clear_round_kernel"] = 1
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
                        "validated+applied (routed to the owner shard over NVLink when G>1); device half of "
                        "mergeCommit (write-set records + devShadow refresh) in every step",
            "stmr_words_per_gpu": W, "batch_tx": B, "log_entries_per_gpu": L, "rs_gran_bytes": args.gran,
            "stmr_layout": "16-B word cells {value, lock-or-TS}", "parallelism": f"shard{world}",
            "log_exchange": exchange,
            "step": "executeBatch -> validateChunk(apply) -> merge_stage -> clearRound",
            "l2": "inputs larger than L2: 1 GiB STMR per GPU, rotating per-step input buffers "
                  f"({n_bufs} tx batches + {n_steps} logs, {(n_bufs * B * 24 + n_steps * L * 24) >> 20} MiB)",
        },
        "roofline": {"bound": "hbm", "kernel": "bank_batch_kernel", "achieved": achieved, "peak": peak,
                     "peak_kind": peak_kind, "unit": "GB/s", "frac": achieved / peak,
                     "peak_nominal": NOMINAL_HBM_GBS, "frac_nominal": achieved / NOMINAL_HBM_GBS,
                     "traffic": measured_traffic("bank_batch_kernel"),
                     "traffic_source": "profiles/traffic.json (ncu --set full, dram read+write per launch)",
                     "algorithmic_bytes_per_tx": TX_BYTES, "kernel_ms": batch_ms,
                     "kernel_share_of_step": batch_ms / ms_step,
                     "protocol_floor": protocol_floor(batch_ms, measured_traffic("bank_batch_kernel"), peak)},
        "step_breakdown_ms": {"batch": batch_ms, "validate_apply": val_ms, "merge_stage": mstage_ms,
                              "step": ms_step},
        "validate_apply_cfg2": {"kernel": "apply_xchg_kernel", "gbs_algorithmic": val_gbs,
                                "entries_per_s_per_gpu": (n_val / K / world) / (val_ms / 1e3),
                                "frac": val_gbs / peak, "algorithmic_bytes_per_entry": ENTRY_BYTES,
                                "traffic": measured_traffic("validate_apply"), "kernel_ms": val_ms},
        "batch": {"committed_last": int(st.committed), "aborts_last": int(st.aborts)},
        "bank_sum_ok": bank_sum_ok, "shadow_equals_replica": shadow_ok,
        "e2e": e2e,
        "gpu_launches": K * launches_per_step,
        "gpu_launches_per_step": launches_detail,
        "clocks": clk.summary(),
        "input_gen_s": gen_s,
    }
    dev.close()
    host_replica.free()
    torch.cuda.synchronize()
    torch.cuda.empty_cache()

    if rank == 0 and world == 1 and args.live_rounds > 0:
        line["e2e_live"] = run_live(args)
    if world == 1 and not args.no_configs:
        line["configs"] = run_configs(args, hetm, torch)
    if not args.no_cfg5:
        line["validate_apply"] = run_cfg5(args, hetm, torch, world, rank, local, dist, peak)
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(args, seconds=args.cpu_seconds)
    if rank == 0:
        print(json.dumps(line), flush=True)
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
    dev.sync()
    dev.read_counters()
    dev.clear_round()  # synchronous clear: refresh the TS floor after the pipelined rounds
    # the device-timed loop staged its merges without shipping them: realign the
    # host replica's device half first (raw read under quiescence)
    host_replica.array[:W // 2] = dev.download(hetm.REPLICA_DEV, base, W // 2)
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
        dt = max_over_ranks(dist, [dt])[0]
    # the host replica holds the host's own commits on its half; the device half must match the device
    dev_half = dev.download(hetm.REPLICA_DEV, base, W // 2)
    replica_ok = bool((host_replica.array[:W // 2] == dev_half).all())
    for p in txs + logs + [tickets]:
        p.free()
    return {"value": world * B * steps / dt, "unit": UNIT, "h2d_bytes_per_step": h2d // steps,
            "d2h_bytes_per_step": d2h // steps, "steps": steps, "ms_per_step": dt / steps * 1e3,
            "host_replica_matches_device": replica_ok,
            "merge": ("chunk copy (SPEC.md:363-371)" if args.chunk_merge else
                      "delta (12-B {word,value} per device-written word)" +
                      (", staged + speculatively applied right after the execution phase (hetm_dev_merge_prepare)"
                       if args.early_merge else "")),
            "bound": "host DRAM: the merge scatter of ~2^21 random words into the host replica per round plus "
                     "the DMAs (profiles/r01_e2e_bounds.txt)",
            "timing": "host wall clock around full rounds (pinned buffers; verdict + merge D2H landed in the host "
                      "replica before the next round's host log; the next GPU batch overlaps the merge, PAPER.md:355)"}


def run_live(args):
    """e2e with a LIVE producer: Engine::runRound at
    configs[1] scale, TL2 host workers committing on the host half while the
    GPU runs the batch; hostCutoff 4, early validation every 8 chunks."""
    exe = os.path.join(ROOT, "build", "hetm_live_round")
    if not os.path.exists(exe):
        return {"error": "build/hetm_live_round not built (run __graft_entry__.build())"}
    cmd = [exe, str(args.live_rounds), str(args.words_log2), str(args.batch)]
    try:
        out = subprocess.run(cmd, capture_output=True, text=True, timeout=300)
    except subprocess.TimeoutExpired:
        return {"error": "timeout"}
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    if out.returncode != 0 or not lines:
        return {"error": f"rc {out.returncode}: {(out.stdout + out.stderr)[-400:]}"}
    r = json.loads(lines[-1])
    r.update({"value": r["tx_per_s"], "unit": "tx/s (host + device commits)", "driver": "build/hetm_live_round",
              "timing": "host wall clock over full rounds (first round warm-up); host replica and device batch "
                        "inputs in pinned host memory, logs streamed through the pinned staging ring"})
    return r


def _device_rounds_time(fn, rounds, torch):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    res = [fn(r) for r in range(rounds)]
    torch.cuda.synchronize()
    return time.perf_counter() - t0, res


def run_configs(args, hetm, torch):
    """BASELINE configs[2] and [3] on one GPU, device-resident inputs."""
    out = {}
    B = args.batch
    R = args.config_rounds
    # ---- configs[2]: zipf 0.99 on both sides over the same 1 GiB STMR -> conflict
    # every round unless the starvation guard (K = 3) makes the
    # host read-only; FavorHost: DeviceAborted -> optimized mergeAbortDevice.
    W = 1 << args.words_log2
    d = hetm.GpuDevice(W, rs_gran_bytes=args.gran, log_capacity=B, merge_delta=True)
    d.register_kernel(hetm.KERNEL_BANK)
    d.upload(hetm.REPLICA_DEV, 0, np.full(W, 1000, np.uint64))
    d.merge_commit(np.full(W, 1000, np.uint64))
    d.merge_wait()
    d.clear_round()
    bats = [torch.from_numpy(hetm.gen_bank_batch(60 + k, B, 0, W, zipf=0.99).view(np.uint8)).cuda() for k in range(2)]
    logs = []
    for r in range(R + 1):
        lg = hetm.gen_host_log(70 + r, B // 2, 2, 8, 0, W, ts_base=(r + 1) << 32, zipf=0.99)
        logs.append(torch.from_numpy(lg.view(np.uint64).reshape(-1, 3).astype(np.int64)).cuda())
    tk = torch.empty(B, dtype=torch.int64, device="cuda")
    K_GUARD = 3
    state = {"aborts_in_row": 0}

    def zipf_round(r):  # r = -1: warm-up
        guard = state["aborts_in_row"] >= K_GUARD  # read-only host round: no write log
        d.execute_batch_dptr(hetm.KERNEL_BANK, bats[r % 2].data_ptr(), B, tk.data_ptr())
        if not guard:  # logs[r + 1]: ts monotone across the warm-up and the timed rounds
            lg = logs[r + 1]
            d.validate_dptr(lg.data_ptr(), lg.shape[0], hetm.APPLY | hetm.RETAIN)
        conflict = d.round_verdict()
        _, st = d.read_counters()
        if conflict:
            d.merge_abort_device(None, optimized=True)
            state["aborts_in_row"] += 1
        else:
            d.merge_stage()
            state["aborts_in_row"] = 0
        d.clear_round()
        return conflict, int(st.committed), int(st.aborts)

    zipf_round(-1)  # warm-up: a conflicting round (also builds the SCAN graph) ...
    state["aborts_in_row"] = K_GUARD
    zipf_round(-1)  # ... and a read-only host round, which commits (sizes the merge buffers)
    state["aborts_in_row"] = 0
    dt, res = _device_rounds_time(zipf_round, R, torch)
    committed = sum(c for conflict, c, _ in res if not conflict)
    out["cfg3_zipf"] = {
        "workload": "BASELINE configs[2]: bank 2^20-tx batches, accounts zipf(0.99) over the whole 1 GiB STMR; "
                    "host log 2^20 entries zipf(0.99) over the same range -> conflict; FavorHost, optimized "
                    "rollback, starvation guard K=3 (read-only host round after 3 device aborts)",
        "value": committed / dt, "unit": "committed GPU tx/s", "rounds": R, "ms_per_round": dt / R * 1e3,
        "device_aborted_rounds": sum(1 for c, _, _ in res if c),
        "batch_aborted_attempts": sum(a for _, _, a in res),
        "schedule": "AUTO (hot batch -> SCAN)",
        "timing": "host wall clock, device-resident inputs; verdict read and rollback synchronous every round"}
    d.close()
    del bats, logs
    torch.cuda.empty_cache()

    # ---- configs[3]: MemcachedGPU-style cache, 2^20 sets x 8 ways, GET/SET 90/10,
    # keys zipf(0.5) over 4 M keys on the GPU's half (last key bit)
    n_sets = 1 << 20
    Wc = n_sets * 64
    d = hetm.GpuDevice(Wc, rs_gran_bytes=args.gran, merge_delta=True)
    d.register_kernel(hetm.KERNEL_CACHE)
    d.merge_commit(np.zeros(Wc, np.uint64))
    d.merge_wait()
    d.clear_round()
    res_t = torch.empty(B * 40, dtype=torch.uint8, device="cuda")
    warm = torch.from_numpy(hetm.gen_cache_batch(1, B, 1 << 22, 0.5, get_permille=0, part=1).view(np.uint8)).cuda()
    d.execute_batch_dptr(hetm.KERNEL_CACHE, warm.data_ptr(), B, tk.data_ptr(), 0, res_t.data_ptr())
    d.merge_stage()
    d.clear_round()
    cb = [torch.from_numpy(hetm.gen_cache_batch(10 + k, B, 1 << 22, 0.5, get_permille=900, part=1).view(np.uint8)).cuda()
          for k in range(4)]

    def cache_round(r):
        d.execute_batch_dptr(hetm.KERNEL_CACHE, cb[r % 4].data_ptr(), B, tk.data_ptr(), 0, res_t.data_ptr())
        d.merge_stage()
        d.clear_round(asynchronous=True)
        return 0

    cache_round(0)
    d.sync()
    d.set_timing(True)
    d.timing(0)
    dt, _ = _device_rounds_time(cache_round, R, torch)
    bt, bc = d.timing(0)
    d.set_timing(False)
    _, st = d.read_counters()
    out["cfg4_cache"] = {
        "workload": "BASELINE configs[3]: set-associative cache 2^20 sets x 8 ways x 64 B in the STMR (512 MiB), "
                    "2^20 GET/SET per batch 90/10, keys zipf(0.5) over 4 M keys on the GPU's half",
        "value": B * R / dt, "unit": "committed GPU tx/s", "rounds": R, "ms_per_round": dt / R * 1e3,
        "batch_kernel_ms": bt / max(bc, 1), "batch_tx_per_s": B / (bt / max(bc, 1) * 1e-3),
        "schedule": "AUTO (>= 8192 tx -> SCAN: sort by set, one thread per set segment)",
        "timing": "host wall clock over pipelined device rounds (batch + merge_stage + async clear), "
                  "device-resident inputs"}
    d.close()
    del cb, warm, res_t, tk
    torch.cuda.empty_cache()
    return out


def run_cfg5(args, hetm, torch, world, rank, local, dist, peak):
    """BASELINE configs[4]: validate + apply of global CPU write logs over a
    sharded STMR (64 GiB over G GPUs).  Each rank ingests 1/G of the global log
    (uniform over all 2^33 words); at G > 1 the fused route kernel stores every
    entry into its owner's receive arena over NVLink (PeerValidator), a device
    barrier, then every owner validates + applies what it received.  Times are
    CUDA events on the validation stream around route + exchange + apply, max
    over ranks."""
    from paper_1905_00661_b200.shard import PeerValidator

    plan = cfg5_plan(args, world)
    Wg = plan["stmr_words_global"]
    Ws = plan["shard_words"]
    base = rank * Ws
    d = hetm.GpuDevice(Ws, shard_base=base, rs_gran_bytes=1024, device=local, shadow=False, log_capacity=1 << 20)
    s_val = d.stream_handle(2)
    vs = torch.cuda.ExternalStream(s_val)
    # RS bitmap at density 1e-3 of its bits, seeded per shard
    nbits = Ws * 8 // 1024
    rng = np.random.default_rng(1234 + rank)
    bits = rng.integers(0, nbits, max(1, nbits // 1000)).astype(np.uint64)
    rs = np.zeros((nbits + 63) // 64, np.uint64)
    np.bitwise_or.at(rs, (bits >> np.uint64(6)).astype(np.int64), np.left_shift(np.uint64(1), bits & np.uint64(63)))
    n_max = max(s["entries_ingested_per_rank"] for s in plan["sizes"])
    pv = None
    exchange = "none (1 shard)"
    if world > 1:
        pv = PeerValidator(d, world, rank, Ws, n_max, dist, s_val)
        exchange = "fused route kernel -> NVLink peer stores into the owner's arena (CUDA IPC); NCCL 4-B device barrier"
    g = torch.Generator(device="cuda").manual_seed(99 + rank)
    log = torch.empty((n_max, 3), dtype=torch.int64, device="cuda")
    ts_next = 1
    rows = []
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for sz in plan["sizes"]:
        n = sz["entries_ingested_per_rank"]
        lg = log[:n]
        lg[:, 0] = torch.randint(0, Wg, (n,), device="cuda", generator=g)
        lg[:, 1] = torch.randint(-(1 << 62), 1 << 62, (n,), device="cuda", generator=g)
        times = []
        for r in range(args.cfg5_reps + 1):
            d.clear_round()  # rolls the TS floor: every rep is a fresh round
            d.or_bitmap(hetm.BMP_RS, rs)
            # globally unique, monotone ts: rank-interleaved
            lg[:, 2] = torch.arange(ts_next, ts_next + n, device="cuda", dtype=torch.int64) * world + rank
            ts_next += n
            torch.cuda.synchronize()
            if dist:
                dist.barrier()
            ev0.record(vs)
            if pv is not None:
                with torch.cuda.stream(vs):
                    pv.validate(lg, hetm.APPLY)
            else:
                d.validate_dptr(lg.data_ptr(), n, hetm.APPLY, s_val)
            ev1.record(vs)
            torch.cuda.synchronize()
            if r:
                times.append(ev0.elapsed_time(ev1))
        ms = max_over_ranks(dist, [statistics.median(times)])[0]
        conflict = d.round_verdict()
        n_glob = sz["entries_global"]
        gbs = ENTRY_BYTES * n_glob / (ms * 1e-3) / 1e9
        rows.append({**sz, "ms": ms, "entries_per_s": n_glob / (ms * 1e-3), "gbs_algorithmic": gbs,
                     "frac": gbs / (world * peak), "frac_nominal": gbs / (world * NOMINAL_HBM_GBS),
                     "log_gbs": LOG_ENTRY_WIRE * n_glob / (ms * 1e-3) / 1e9, "conflict": bool(conflict)})
    if pv is not None:
        pv.close()
    d.close()
    del log
    torch.cuda.empty_cache()
    head = next((r for r in rows if r["log_mib_global"] == 1024), rows[-1])
    return {"workload": f"BASELINE configs[4]: {plan['stmr_gib_global']:.0f} GiB STMR sharded {plan['shard_gib']:.0f} "
                        f"GiB per GPU (no shadow), global CPU write logs uniform over the STMR, RS density 1e-3 at "
                        "1 KiB granules",
            "n_gpus": world, "exchange": exchange, "kernel": "apply_xchg_kernel (+ route_peer_scatter_kernel at G>1)",
            "headline_log_mib": head["log_mib_global"], "gbs_algorithmic": head["gbs_algorithmic"],
            "aggregate_gbs": head["gbs_algorithmic"], "frac": head["frac"], "peak_per_gpu": peak,
            "algorithmic_bytes_per_entry": ENTRY_BYTES, "entries_per_s": head["entries_per_s"],
            "sweep": rows, "geometry": {k: v for k, v in plan.items() if k != "sizes"},
            "timing": "CUDA events on the validation stream around route + NVLink delivery + apply, median of "
                      f"{args.cfg5_reps} reps, max over ranks"}


# ---------------------------------------------------------- CPU baseline
def cpu_baseline(args, seconds=8.0, rounds=None):
    """The reference CPU path (oracle port, multi-threaded) on the SAME round as
    the GPU step: one 2^20-tx bank batch (guest-stm-batch worker pool,
    SPEC.md:237) + validate/apply of the round's 2^20-entry log
     on all host threads, 2^27-word STMR."""
    import oracle as O

    threads = os.cpu_count() or 1
    W = 1 << args.words_log2
    B = args.batch
    L = args.log_entries
    s = np.full(W, 1000, np.uint64)
    ts = np.zeros(W, np.uint64)
    gran = args.gran
    done_tx, t_tot, t_val, r = 0, 0.0, 0.0, 0
    while (rounds is None and (t_tot < seconds or r < 2)) or (rounds is not None and r < rounds):
        txs = O.gen_bank_batch(3000 + r, B, 0, W // 2)
        log = O.gen_host_log(4000 + r, L // 2, 2, 8, W // 2, W // 2, ts_base=r * L)
        t0 = time.perf_counter()
        c, _, rsb, _, _ = O.mt_bank_batch(s, txs, threads, lock_entries=1 << 24, gran=gran, tickets=False)
        t1 = time.perf_counter()
        O.mt_validate_apply(log, rsb, gran, ts, s, threads)
        t2 = time.perf_counter()
        t_tot += t2 - t0
        t_val += t2 - t1
        done_tx += c
        r += 1
    return {"value": done_tx / t_tot, "unit": UNIT, "cores": threads, "kind": "port",
            "sample": f"{r} full rounds x ({B} bank tx + {L} log entries) on the 2^{args.words_log2}-word STMR "
                      "(the GPU step's configuration), oracle/hetm_oracle.c pthreads",
            "validate_apply_entries_per_s": r * L / t_val, "rounds": r, "ms_per_round": t_tot / r * 1e3,
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
    import oracle  # noqa: F401  (builds the checker if needed)
    cpu_baseline(args, rounds=max(1, min(args.warmup, 3)))  # warm-up rounds, untimed
    t0 = time.perf_counter()
    cb = cpu_baseline(args, rounds=args.steps)
    dt = time.perf_counter() - t0
    line = {"metric": METRIC, "value": cb["value"], "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": dt / args.steps * 1e3, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "u64", "data": "synthetic",
            "impl": "reference",
            "config": {"workload": "BASELINE configs[1]: one full round per step (2^20 bank tx + 2^20 log "
                                   "entries, 2^27-word STMR), identical to the GPU arm's step",
                       "stmr_words": 1 << args.words_log2, "batch_tx": args.batch,
                       "log_entries": args.log_entries},
            "cpu_baseline": cb,
            "e2e": {"value": cb["value"], "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def run_plan(args):
    """Configuration line without GPU work: exercises the rank spawn and the
    process group (gloo on CPU), reports the geometry and NVLink byte counts."""
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group(os.environ.get("HETM_BENCH_BACKEND", "gloo"))
        import torch
        t = torch.ones(1)
        dist.all_reduce(t)
        assert int(t.item()) == world
    line = {"metric": METRIC, "plan": True, "n_gpus": world, "rank_count_checked": world,
            "config": {"stmr_words_per_gpu": 1 << args.words_log2, "batch_tx": args.batch,
                       "log_entries_per_gpu": args.log_entries, "parallelism": f"shard{world}"},
            "validate_apply": cfg5_plan(args, world)}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if dist:
        dist.barrier()
        dist.destroy_process_group()


def main():
    args = parse()
    maybe_spawn(args)
    if args.plan:
        run_plan(args)
    elif args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
