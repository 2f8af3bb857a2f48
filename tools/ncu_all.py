"""Exercise every product kernel of libhetm_b200.so once at a representative
size, for one `ncu --set full` capture of all of them (profiles/r02_ncu_*):

  ncu --set full --clock-control none --import-source on -o gpurun_out/all \
      python tools/ncu_all.py

Shapes: BASELINE configs[1] (2^27-word shard, 2^20-tx bank batch, 2^20-entry
host log), the cache of configs[3] (2^20 sets, 2^20 GET/SET), a 4-shard route,
and a 2-handle bitmap OR / peer delivery on one GPU (the multi-GPU kernels'
code path with plain device pointers instead of NVLink peer pointers).  Product
generators only (no oracle)."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_1905_00661_b200 as hetm  # noqa: E402

W = 1 << 27
B = 1 << 20
L = 1 << 20


def cuda_log(seed, n_tx, lo, span, ts_base):
    lg = hetm.gen_host_log(seed, n_tx, 2, 8, lo, span, ts_base=ts_base)
    return torch.from_numpy(lg.view(np.uint64).reshape(-1, 3).astype(np.int64)).cuda()


def bank_round():
    d = hetm.GpuDevice(W, rs_gran_bytes=1024, merge_delta=True, log_capacity=L)
    d.register_kernel(hetm.KERNEL_BANK)
    init = np.full(W, 1000, np.uint64)
    d.upload(hetm.REPLICA_DEV, 0, init)                      # scatter_range_kernel
    host = hetm.PinnedArray((W,), np.uint64)
    host.array[:] = init
    d.merge_commit(host.array)                              # dirty_chunks_kernel (full shadow)
    d.merge_wait()
    d.clear_round()
    tx = torch.from_numpy(hetm.gen_bank_batch(1, B, 0, W // 2).view(np.uint8)).cuda()
    tickets = torch.empty(B, dtype=torch.int64, device="cuda")
    d.set_schedule(hetm.SCHED_OPTIMISTIC)
    d.execute_batch_dptr(hetm.KERNEL_BANK, tx.data_ptr(), B, tickets.data_ptr())   # bank_batch_kernel
    lg = cuda_log(2, L // 2, W // 2, W // 2, 0)
    d.validate_dptr(lg.data_ptr(), L, hetm.VALIDATE_ONLY)    # validate_kernel
    d.validate_dptr(lg.data_ptr(), L, hetm.APPLY | hetm.RETAIN)  # apply_kernel + restore_kernel
    d.merge_stage()                                         # delta_pick + delta_emit + shadow_sync
    d.merge_commit(host.array)
    d.merge_wait()
    d.clear_round()                                         # clear_round_kernel
    # SCAN schedule of a zipf batch: keys, the hand-written radix sort, commit
    d.set_schedule(hetm.SCHED_SCAN)
    tz = torch.from_numpy(hetm.gen_bank_batch(3, B, 0, W // 2, zipf=0.99).view(np.uint8)).cuda()
    d.execute_batch_dptr(hetm.KERNEL_BANK, tz.data_ptr(), B, tickets.data_ptr())   # sched_* + sort_*
    d.sync()
    # a conflicting round: host log over the device's accounts -> optimized rollback
    lc = cuda_log(4, L // 2, 0, W // 2, L)
    d.validate_dptr(lc.data_ptr(), L, hetm.APPLY | hetm.RETAIN)
    assert d.round_verdict()
    d.merge_abort_device(None, optimized=True)              # wlog_restore + untag + apply + log_to_shadow
    d.clear_round()
    d.download(hetm.REPLICA_DEV, 0, 1 << 20)                # gather_range_kernel
    d.close()
    host.free()


def traced_batches():
    Wt = 1 << 20
    d = hetm.GpuDevice(Wt, rs_gran_bytes=1024)
    d.register_kernel(hetm.KERNEL_BANK)
    d.upload(hetm.REPLICA_DEV, 0, np.full(Wt, 1000, np.uint64))
    n = 1 << 16
    for sched in (hetm.SCHED_OPTIMISTIC, hetm.SCHED_SCAN):  # KO_TRACE bank kernel; traced SCAN (segmented scan)
        d.set_schedule(sched)
        out = np.zeros(n * hetm.TRACE_TX_WORDS, np.uint64)
        d.trace_next_batch(out)
        d.execute_batch(hetm.KERNEL_BANK, hetm.gen_bank_batch(5 + sched, n, 0, Wt))
        d.sync()
        d.clear_round()
    d.register_kernel(hetm.KERNEL_RW)
    rw = np.zeros(n, hetm.RW_TX)
    rng = np.random.default_rng(6)
    for f in rw.dtype.names:
        if rw.dtype[f].kind == "u" and rw.dtype[f].shape == ():
            rw[f] = rng.integers(0, Wt, n)
    try:
        d.execute_batch(hetm.KERNEL_RW, rw)                  # rw_batch_kernel (generic TM_read/TM_write)
    except Exception as e:  # noqa: BLE001 - the record layout is the test suite's business
        print("rw batch skipped:", e)
    d.sync()
    d.close()


def cache_batches():
    n_sets = 1 << 20
    Wc = n_sets * hetm.CACHE_SET_WORDS
    d = hetm.GpuDevice(Wc, rs_gran_bytes=1024)
    d.register_kernel(hetm.KERNEL_CACHE)
    d.set_cache_geometry(0, n_sets)
    for n in (4096, 1 << 20):                               # optimistic cache_batch_kernel; SCAN cs_* + select
        d.execute_batch(hetm.KERNEL_CACHE, hetm.gen_cache_batch(7, n, 4 << 20, 0.5, 900, 1))
        d.sync()
    d.close()


def shards_and_peers():
    G, Ws = 4, 1 << 24
    devs = [hetm.GpuDevice(Ws, shard_base=s * Ws, rs_gran_bytes=1024) for s in range(G)]
    lg = cuda_log(8, L // 2, 0, G * Ws, 10 * L)
    out = torch.empty_like(lg)
    counts = torch.zeros(64, dtype=torch.int64, device="cuda")
    devs[0].route_log_dptr(lg.data_ptr(), L, G, Ws, out.data_ptr(), counts.data_ptr())   # route_count/scan/scatter
    cap = L
    arenas = [d.recv_arena(G, cap) for d in devs]
    devs[0].route_to_peers_dptr(lg.data_ptr(), L, G, Ws, 0, cap, 0, [a[0] for a in arenas],
                                [a[1] for a in arenas])     # route_peer_publish + route_peer_scatter
    for d in devs:
        d.sync()
    devs[1].apply_received(0, hetm.APPLY)                   # apply over the received regions
    d0, d1 = devs[0], devs[1]
    d0.register_kernel(hetm.KERNEL_BANK)
    d0.execute_batch(hetm.KERNEL_BANK, hetm.gen_bank_batch(9, 1 << 16, 0, Ws))
    d0.sync()
    d1.bitmap_or_peers(hetm.BMP_RS, [d0.bitmap_dptr(hetm.BMP_RS)[0]])   # or_peers_kernel
    d1.or_bitmap(hetm.BMP_WS, d0.snapshot(hetm.BMP_WS).words)           # or_words_kernel
    d1.bitmap_stats()                                                   # popcount_kernel
    d1.sync()
    for d in devs:
        d.close()


def chunk_merge():
    d = hetm.GpuDevice(W, rs_gran_bytes=1024, log_capacity=L)      # SPEC chunk form of mergeCommit
    d.register_kernel(hetm.KERNEL_BANK)
    host = hetm.PinnedArray((W,), np.uint64)
    host.array[:] = 0
    d.execute_batch(hetm.KERNEL_BANK, hetm.gen_bank_batch(10, 1 << 18, 0, W // 2))
    d.round_verdict()
    d.merge_commit(host.array)                              # dirty_chunks_kernel (incremental shadow)
    d.merge_wait()
    d.close()
    host.free()


if __name__ == "__main__":
    for f in (bank_round, traced_batches, cache_batches, shards_and_peers, chunk_merge):
        f()
        torch.cuda.synchronize()
        print("done", f.__name__, flush=True)
