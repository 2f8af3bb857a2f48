"""Bank batch schedules (capi.h HETM_SCHED_*) vs the CPU oracle.

OPTIMISTIC (PR-STM-style phased kernel) and SCAN (sort + segmented scan in
input order, bank_sched.cu) must both give batches whose ticket-order replay
on the oracle reproduces the STMR, RS / WS / ChunkMap and the write-set log
(the delta merge) bit-exactly; SCAN additionally commits in input order with
no aborts, and AUTO picks it for hot host batches only.
"""
import numpy as np
import pytest

from test_gpu_parity import check_replay, dev_factory  # noqa: F401  (fixture)

pytestmark = pytest.mark.gpu


def scheds(hetm):
    return {"optimistic": hetm.SCHED_OPTIMISTIC, "scan": hetm.SCHED_SCAN}


def workload(orc, kind, W, n, seed):
    if kind == "uniform":
        return orc.gen_bank_batch(seed, n, 0, W)
    if kind == "zipf":
        return orc.gen_bank_batch(seed, n, 0, W, zipf=0.99)
    rng = np.random.default_rng(seed)  # duplicate accounts inside records (last write wins)
    t = np.zeros(n, orc.BANK_TX)
    t["acct"] = rng.integers(0, min(W, 16), (n, 4))
    t["amount"] = rng.integers(1, 100, n)
    return t


@pytest.mark.parametrize("sched", ["optimistic", "scan"])
@pytest.mark.parametrize("gran", [8, 1024])
@pytest.mark.parametrize("kind,W,n", [("uniform", 1 << 16, 1 << 15), ("zipf", 1 << 16, 1 << 14),
                                      ("dups", 256, 6000), ("uniform", 64, 1 << 12)])
def test_schedules_replay_bit_exact(hetm, orc, dev_factory, sched, gran, kind, W, n):
    d = dev_factory(W, rs_gran_bytes=gran)
    d.register_kernel(hetm.KERNEL_BANK)
    d.set_schedule(scheds(hetm)[sched])
    init = (np.arange(W, dtype=np.uint64) * np.uint64(977)) % np.uint64(50_000) + np.uint64(10_000)
    d.upload(hetm.REPLICA_DEV, 0, init)
    txs = workload(orc, kind, W, n, W + n)
    r = d.execute_batch(hetm.KERNEL_BANK, txs)
    assert r.committed == n and r.livelocked == 0
    check_replay(hetm, orc, d, txs, r.tickets, init, gran, 16384)
    if sched == "scan":  # input order, nothing aborted
        assert r.aborts == 0
        assert (r.tickets == r.ticket_first + np.arange(n, dtype=np.uint64)).all()


@pytest.mark.parametrize("sched", ["optimistic", "scan"])
def test_schedules_consecutive_batches_and_delta_merge(hetm, orc, dev_factory, sched):
    """Several batches per round (tickets keep increasing), then the delta mergeCommit
    built from the write-set log lands the device writes in the host replica."""
    W = 1 << 18
    d = dev_factory(W, rs_gran_bytes=1024, merge_delta=True)
    d.register_kernel(hetm.KERNEL_BANK)
    d.set_schedule(scheds(hetm)[sched])
    host = np.full(W, 1000, np.uint64)
    d.upload(hetm.REPLICA_DEV, 0, host)
    d.merge_commit(host)
    d.merge_wait()
    d.clear_round()
    ref = host.copy()
    last = -1
    for b in range(3):
        txs = orc.gen_bank_batch(40 + b, 1 << 14, 0, W // 2, zipf=0.99 if b == 1 else 0.0)
        r = d.execute_batch(hetm.KERNEL_BANK, txs)
        assert int(r.tickets.min()) > last
        last = int(r.tickets.max())
        orc.bank_replay(ref, txs, orc.order_by_ticket(r.tickets), 1024, 16384)
    assert not d.round_verdict()
    d.merge_commit(host)
    d.merge_wait()
    assert (host == ref).all() and (d.download(hetm.REPLICA_DEV) == ref).all()


def test_scan_rejects_out_of_shard_transactions(hetm, orc, dev_factory):
    W, base = 1 << 12, 1 << 12
    d = dev_factory(W, rs_gran_bytes=8, shard_base=base)
    d.register_kernel(hetm.KERNEL_BANK)
    d.set_schedule(hetm.SCHED_SCAN)
    txs = orc.gen_bank_batch(5, 1000, base, W)
    txs["acct"][[3, 500]] = 7  # below the shard
    with pytest.raises(hetm.OutOfBoundsError):
        d.execute_batch(hetm.KERNEL_BANK, txs)


def test_auto_feedback_device_pointer_batches(hetm, orc, dev_factory):
    """Device-pointer batches: the abort count of an optimistic AUTO batch is judged
    when the caller next reads the counters (a verdict or read_counters sync)."""
    import torch

    W, n = 1 << 14, 1 << 14
    d = dev_factory(W, rs_gran_bytes=8)
    d.register_kernel(hetm.KERNEL_BANK)
    init = np.full(W, 1000, np.uint64)
    d.upload(hetm.REPLICA_DEV, 0, init)
    ref = init.copy()
    tk = torch.empty(n, dtype=torch.int64, device="cuda")
    seq = []
    for k in range(3):
        txs = orc.gen_bank_batch(400 + k, n, 0, W)
        b = torch.from_numpy(txs.view(np.uint8)).cuda()
        d.execute_batch_dptr(hetm.KERNEL_BANK, b.data_ptr(), n, tk.data_ptr())
        d.sync()
        _, st = d.read_counters()
        t = tk.cpu().numpy().astype(np.uint64)
        orc.bank_replay(ref, txs, orc.order_by_ticket(t), 8, 16384)
        seq.append((int(st.retried), bool((np.diff(t.astype(np.int64)) == 1).all())))
    assert (d.download(hetm.REPLICA_DEV) == ref).all()
    assert seq[0][0] * 1024 > n and not seq[0][1]         # optimistic, retry-heavy (capi.cu kAutoRetryRatio)
    assert seq[1] == (0, True) and seq[2] == (0, True)    # then SCAN


def test_auto_feedback_host_buffer_batches(hetm, orc, dev_factory):
    """Host-buffer batches: an optimistic AUTO batch whose transactions needed a third
    attempt more than once per 1024 (conflict chains the CPU sample did not flag)
    sends the next batches to SCAN, judged at the end of the call."""
    W, n = 1 << 14, 1 << 14
    d = dev_factory(W, rs_gran_bytes=8)
    d.register_kernel(hetm.KERNEL_BANK)
    init = np.full(W, 1000, np.uint64)
    d.upload(hetm.REPLICA_DEV, 0, init)
    ref = init.copy()
    seq = []
    for k in range(3):
        txs = orc.gen_bank_batch(500 + k, n, 0, W)
        r = d.execute_batch(hetm.KERNEL_BANK, txs)
        orc.bank_replay(ref, txs, orc.order_by_ticket(r.tickets), 8, 16384)
        seq.append((int(r.retried), bool((np.diff(r.tickets.astype(np.int64)) == 1).all())))
    assert (d.download(hetm.REPLICA_DEV) == ref).all()
    assert seq[0][0] * 1024 > n and not seq[0][1]         # optimistic, retry-heavy
    assert seq[1] == (0, True) and seq[2] == (0, True)    # then SCAN


def test_auto_takes_scan_for_hot_batches_only(hetm, orc, dev_factory):
    W, n = 1 << 20, 1 << 16
    d = dev_factory(W, rs_gran_bytes=1024)
    d.register_kernel(hetm.KERNEL_BANK)  # AUTO is the default
    d.upload(hetm.REPLICA_DEV, 0, np.full(W, 1000, np.uint64))
    hot = d.execute_batch(hetm.KERNEL_BANK, orc.gen_bank_batch(1, n, 0, W, zipf=0.99))
    assert hot.aborts == 0 and (np.diff(hot.tickets.astype(np.int64)) == 1).all()
    cold = d.execute_batch(hetm.KERNEL_BANK, orc.gen_bank_batch(2, n, 0, W))
    assert (np.diff(cold.tickets.astype(np.int64)) != 1).any()  # optimistic: commit order != input order


def test_deterministic_mode_runs_scan_in_input_order(hetm, orc, dev_factory):
    W, n = 1 << 14, 1 << 14
    d = dev_factory(W, rs_gran_bytes=8, deterministic=True)
    d.register_kernel(hetm.KERNEL_BANK)
    d.set_schedule(hetm.SCHED_OPTIMISTIC)  # the deterministic mode overrides it for bank batches
    init = np.full(W, 1000, np.uint64)
    d.upload(hetm.REPLICA_DEV, 0, init)
    txs = orc.gen_bank_batch(9, n, 0, W, zipf=0.99)
    r = d.execute_batch(hetm.KERNEL_BANK, txs)
    assert (r.tickets == r.ticket_first + np.arange(n, dtype=np.uint64)).all() and r.aborts == 0
    check_replay(hetm, orc, d, txs, r.tickets, init, 8, 16384)


def test_auto_device_batches_follow_the_previous_estimate(hetm, orc, dev_factory):
    """Device-pointer batches under AUTO: the first hot batch runs optimistic, later ones switch to
    SCAN from the side-stream estimate of an earlier batch; uniform batches never switch."""
    import torch
    W, n = 1 << 16, 1 << 14
    d = dev_factory(W, rs_gran_bytes=1024)
    d.register_kernel(hetm.KERNEL_BANK)
    init = np.full(W, 1000, np.uint64)
    d.upload(hetm.REPLICA_DEV, 0, init)
    tk = torch.empty(n, dtype=torch.int64, device="cuda")

    def run(txs):
        b = torch.from_numpy(txs.view(np.uint8)).cuda()
        d.execute_batch_dptr(hetm.KERNEL_BANK, b.data_ptr(), n, tk.data_ptr())
        d.sync()
        _, st = d.read_counters()
        t = tk.cpu().numpy().view(np.uint64)
        d.clear_round()
        return st, t

    ref = init.copy()
    sts = []
    for k in range(4):
        txs = orc.gen_bank_batch(60 + k, n, 0, W, zipf=0.99)
        st, t = run(txs)
        orc.bank_replay(ref, txs, orc.order_by_ticket(t), 1024, 16384)
        sts.append((st.aborts, bool((np.diff(t.astype(np.int64)) == 1).all())))
    assert (d.download(hetm.REPLICA_DEV) == ref).all()
    assert sts[0][0] > 0                              # first hot batch: optimistic (no estimate yet)
    assert sts[-1] == (0, True)                       # later: SCAN in input order
    # uniform input: back to optimistic once the abort-feedback run (15 batches after the
    # first, abort-heavy hot batch) is over — the estimate itself never flags these
    optimistic_seen = False
    for k in range(20):
        txs = orc.gen_bank_batch(90 + k, n, 0, W)
        st, t = run(txs)
        orc.bank_replay(ref, txs, orc.order_by_ticket(t), 1024, 16384)
        if not (np.diff(t.astype(np.int64)) == 1).all():
            optimistic_seen = True
            break
    assert (d.download(hetm.REPLICA_DEV) == ref).all()
    assert optimistic_seen and k >= 11


@pytest.mark.parametrize("W,n", [(1000, 1), (1000, 3), (12345, 777), (1 << 10, 0)])
def test_scan_edge_sizes(hetm, orc, dev_factory, W, n):
    """Non-power-of-two shards, single transactions and empty batches under SCAN."""
    d = dev_factory(W, rs_gran_bytes=8)
    d.register_kernel(hetm.KERNEL_BANK)
    d.set_schedule(hetm.SCHED_SCAN)
    init = np.arange(W, dtype=np.uint64) + np.uint64(5000)
    d.upload(hetm.REPLICA_DEV, 0, init)
    txs = orc.gen_bank_batch(W + n, n, 0, W) if n else np.zeros(0, orc.BANK_TX)
    r = d.execute_batch(hetm.KERNEL_BANK, txs)
    assert r.committed == n and r.aborts == 0
    if n:
        check_replay(hetm, orc, d, txs, r.tickets, init, 8, 16384)
    else:
        assert (d.download(hetm.REPLICA_DEV) == init).all() and d.bitmap_stats() == (0, 0, 0)


@pytest.mark.parametrize("n", [(1 << 13) - 1, 1 << 13])
def test_cache_auto_threshold_both_sides(hetm, orc, dev_factory, n):
    """AUTO runs cache batches below 8192 optimistic and from 8192 as SCAN; both replay bit-exactly."""
    from test_gpu_parity import check_cache_replay
    n_sets = 1 << 10
    W = n_sets * 64
    d = dev_factory(W, rs_gran_bytes=1024)
    d.register_kernel(hetm.KERNEL_CACHE)
    init = np.zeros(W, np.uint64)
    txs = orc.gen_cache_batch(3, n, n_sets * 4, 0.5, get_permille=500, part=-1, steal_permille=500)
    r = d.execute_batch(hetm.KERNEL_CACHE, txs, results=True)
    check_cache_replay(hetm, orc, d, txs, r, init, n_sets)
    in_order = bool((r.tickets == r.ticket_first + np.arange(n, dtype=np.uint64)).all())
    assert in_order == (n >= 1 << 13) or r.aborts == 0
