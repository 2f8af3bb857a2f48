"""GPU parity: the sm_100a path through the C-ABI vs the CPU oracle.

Bit-exact for everything (all arithmetic on the path is integer).  Sizes are
small enough for the oracle to finish in seconds; tests marked `slow` run the
BASELINE configuration (1 GiB STMR, 2^20-tx batches) through size-independent
properties (ticket-order replay, bank-sum invariant, WS subset RS)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

GRANS = [8, 1024]


@pytest.fixture
def dev_factory(hetm):
    made = []

    def make(W, **kw):
        d = hetm.GpuDevice(W, **kw)
        made.append(d)
        return d

    yield make
    for d in made:
        d.close()


def rw_txs(orc, rows):
    t = np.zeros(len(rows), orc.RW_TX)
    for i, (rd, wr, add) in enumerate(rows):
        t[i]["nr"], t[i]["nw"] = len(rd), len(wr)
        t[i]["r_addr"][: len(rd)] = rd
        t[i]["w_addr"][: len(wr)] = wr
        t[i]["add"][: len(add)] = add
    return t


# ------------------------------------------------------------- stmr module
def test_create_zero_filled(hetm, dev_factory):
    d = dev_factory(8, rs_gran_bytes=8)
    assert (d.download(hetm.REPLICA_DEV) == 0).all()
    assert (d.download(hetm.REPLICA_DEV_SHADOW) == 0).all()


def test_raw_ops(hetm, dev_factory):
    d = dev_factory(64, rs_gran_bytes=8)
    d.raw_write(hetm.REPLICA_DEV, 3, 42)
    assert d.raw_read(hetm.REPLICA_DEV, 3) == 42
    assert d.raw_read(hetm.REPLICA_DEV_SHADOW, 3) == 0  # SPEC.md:60 replicas independent
    with pytest.raises(hetm.OutOfBoundsError):
        d.raw_write(hetm.REPLICA_DEV, 64, 1)
    with pytest.raises(hetm.InvalidArgumentError):
        d.raw_write(hetm.REPLICA_HOST, 0, 1)


def test_kernel_registration_errors(hetm, orc, dev_factory):
    d = dev_factory(64, rs_gran_bytes=8)
    with pytest.raises(hetm.NoImplementationError):
        d.register_kernel(99)
    with pytest.raises(hetm.KernelNotRegisteredError):
        d.execute_batch(hetm.KERNEL_BANK, orc.gen_bank_batch(1, 4, 0, 64))
    d.register_kernel(hetm.KERNEL_BANK)
    with pytest.raises(hetm.InvalidSizeError):
        d.execute_batch(hetm.KERNEL_BANK, np.zeros(3, orc.RW_TX))
    with pytest.raises(hetm.OutOfBoundsError):
        d.execute_batch(hetm.KERNEL_BANK, orc.gen_bank_batch(1, 4, 0, 128))


# ------------------------------------------------------- guest-stm-batch
def test_execute_batch_spec_209(hetm, orc, dev_factory):
    """1 tx reading word 0, writing word 1 @8 B -> RS {0,1}, WS {1}, stats (2,1,1)."""
    d = dev_factory(64, rs_gran_bytes=8)
    d.register_kernel(hetm.KERNEL_RW)
    r = d.execute_batch(hetm.KERNEL_RW, rw_txs(orc, [([0], [1], [0])]))
    assert r.committed == 1
    rs, ws = d.snapshot(hetm.BMP_RS), d.snapshot(hetm.BMP_WS)
    assert rs.set_bits().tolist() == [0, 1] and ws.set_bits().tolist() == [1]
    assert d.bitmap_stats() == (2, 1, 1)


def test_execute_batch_spec_210_disjoint_increments(hetm, orc, dev_factory):
    d = dev_factory(4096, rs_gran_bytes=8)
    d.register_kernel(hetm.KERNEL_RW)
    n = 4096
    r = d.execute_batch(hetm.KERNEL_RW, rw_txs(orc, [([], [i], [1]) for i in range(n)]))
    assert r.committed == n and r.aborts == 0  # all commit in one attempt
    assert (d.download(hetm.REPLICA_DEV) == 1).all()


def test_execute_batch_spec_211_same_word(hetm, orc, dev_factory):
    d = dev_factory(64, rs_gran_bytes=8)
    d.register_kernel(hetm.KERNEL_RW)
    r = d.execute_batch(hetm.KERNEL_RW, rw_txs(orc, [([], [5], [1]), ([], [5], [1])]))
    assert r.committed == 2
    assert d.raw_read(hetm.REPLICA_DEV, 5) == 2


def test_clear_round(hetm, orc, dev_factory):
    d = dev_factory(64, rs_gran_bytes=8)
    d.register_kernel(hetm.KERNEL_RW)
    d.execute_batch(hetm.KERNEL_RW, rw_txs(orc, [([0], [1], [0])]))
    d.clear_round()
    assert d.bitmap_stats() == (0, 0, 0)
    d.execute_batch(hetm.KERNEL_RW, np.zeros(0, orc.RW_TX))
    assert d.bitmap_stats() == (0, 0, 0)
    d.clear_round()
    d.clear_round()  # SPEC.md:220 idempotent
    assert d.bitmap_stats() == (0, 0, 0)


def check_replay(hetm, orc, d, txs, tickets, init, gran, chunk, kind="bank"):
    order = orc.order_by_ticket(tickets)
    assert order.size == txs.size, "every transaction commits (SPEC.md:206)"
    assert len(np.unique(tickets)) == txs.size
    ref = init.copy()
    replay = orc.bank_replay if kind == "bank" else orc.rw_replay
    rs, ws, ch = replay(ref, txs, order, gran, chunk, base=d.shard_base)
    got = d.download(hetm.REPLICA_DEV)
    assert (got == ref).all(), f"{int((got != ref).sum())} words differ from ticket-order replay"
    assert (d.snapshot(hetm.BMP_RS).words == rs).all()
    assert (d.snapshot(hetm.BMP_WS).words == ws).all()
    assert (d.snapshot(hetm.BMP_CHUNK).words == ch).all()
    assert ((ws & ~rs) == 0).all()  # WS subset of RS
    return ref


@pytest.mark.parametrize("gran", GRANS)
@pytest.mark.parametrize("W,n", [(1 << 6, 1 << 12), (1 << 10, 1 << 14), (1 << 16, 1 << 16), (1 << 20, 1 << 18)])
def test_bank_batch_replays_in_ticket_order(hetm, orc, dev_factory, gran, W, n):
    d = dev_factory(W, rs_gran_bytes=gran)
    d.register_kernel(hetm.KERNEL_BANK)
    init = np.full(W, 1000, np.uint64)
    d.upload(hetm.REPLICA_DEV, 0, init)
    txs = orc.gen_bank_batch(W + n, n, 0, W)
    r = d.execute_batch(hetm.KERNEL_BANK, txs)
    assert r.committed == n and r.livelocked == 0
    ref = check_replay(hetm, orc, d, txs, r.tickets, init, gran, 16384)
    assert int(ref.sum(dtype=np.uint64)) == 1000 * W  # bank-sum invariant


def test_bank_batch_duplicate_accounts(hetm, orc, dev_factory):
    """Records naming one account twice follow the oracle's sequential semantics."""
    W = 256
    d = dev_factory(W, rs_gran_bytes=8)
    d.register_kernel(hetm.KERNEL_BANK)
    rng = np.random.default_rng(21)
    txs = np.zeros(6000, orc.BANK_TX)
    txs["acct"] = rng.integers(0, 16, (6000, 4))  # many repeats inside a record
    txs["amount"] = rng.integers(1, 100, 6000)
    init = np.full(W, 10_000, np.uint64)
    d.upload(hetm.REPLICA_DEV, 0, init)
    r = d.execute_batch(hetm.KERNEL_BANK, txs)
    assert r.committed == txs.size
    check_replay(hetm, orc, d, txs, r.tickets, init, 8, 16384)


def test_rw_batch_high_contention_replay(hetm, orc, dev_factory):
    W = 64
    d = dev_factory(W, rs_gran_bytes=8)
    d.register_kernel(hetm.KERNEL_RW)
    rng = np.random.default_rng(2)
    rows = []
    for _ in range(20000):
        nr, nw = int(rng.integers(0, 5)), int(rng.integers(1, 3))
        rows.append((rng.integers(0, W, nr).tolist(), rng.integers(0, W, nw).tolist(),
                     rng.integers(0, 100, nw).tolist()))
    txs = rw_txs(orc, rows)
    init = rng.integers(0, 1000, W).astype(np.uint64)
    d.upload(hetm.REPLICA_DEV, 0, init)
    r = d.execute_batch(hetm.KERNEL_RW, txs)
    assert r.committed == 20000
    check_replay(hetm, orc, d, txs, r.tickets, init, 8, 16384, kind="rw")


def test_batches_accumulate_tickets(hetm, orc, dev_factory):
    W = 1 << 12
    d = dev_factory(W, rs_gran_bytes=64)
    d.register_kernel(hetm.KERNEL_BANK)
    init = np.full(W, 7, np.uint64)
    d.upload(hetm.REPLICA_DEV, 0, init)
    ref = init.copy()
    last = 0
    for b in range(3):
        txs = orc.gen_bank_batch(100 + b, 5000, 0, W)
        r = d.execute_batch(hetm.KERNEL_BANK, txs)
        assert r.ticket_first == last and r.tickets.min() >= last
        last = r.ticket_end
        orc.bank_replay(ref, txs, orc.order_by_ticket(r.tickets), 64, 16384)
    assert (d.download(hetm.REPLICA_DEV) == ref).all()


# ------------------------------------------------------------- validation
def random_log(rng, n, W, lo=0, ts0=0, dup_words=None):
    e = np.zeros(n, dtype=[("addr", "<u8"), ("value", "<u8"), ("ts", "<u8")])
    e["addr"] = rng.integers(0, dup_words or W, n) + lo
    e["value"] = rng.integers(0, 2**63, n, dtype=np.uint64)
    e["ts"] = rng.permutation(n) + 1 + ts0
    return e


@pytest.mark.parametrize("gran", GRANS)
def test_validate_apply_matches_oracle(hetm, orc, dev_factory, gran):
    W = 1 << 14
    rng = np.random.default_rng(gran)
    d = dev_factory(W, rs_gran_bytes=gran)
    nbits = W * 8 // gran
    rs = np.zeros((nbits + 63) // 64, np.uint64)
    for b in rng.choice(nbits, 3, replace=False):
        rs[b >> 6] |= np.uint64(1 << int(b & 63))
    d.or_bitmap(hetm.BMP_RS, rs)
    log = random_log(rng, 50000, W, dup_words=512)  # duplicate-heavy
    chunks = np.array_split(log, 16)
    for k in rng.permutation(16):
        d.stream_chunk(chunks[k], src_thread=int(k % 4), seq=int(k))
    conflict = d.round_verdict()
    ts, dev = np.zeros(W, np.uint64), np.zeros(W, np.uint64)
    want = orc.validate_chunk(log, rs, gran, ts, dev)
    assert conflict == want == orc.brute_force_intersect(log, rs, nbits, gran)
    assert (d.download(hetm.REPLICA_DEV) == dev).all()


def test_validate_hot_words_one_chunk(hetm, orc, dev_factory):
    """Many entries per word inside ONE apply launch, ts ascending with the
    entry index (most TS raises race with an earlier entry of the launch): the
    apply kernel's restore queue, and its overflow fallback (> 2^20 raced
    entries), must still leave the freshest value in every word."""
    W = 1 << 12
    for n, tsorder in ((1 << 16, "random"), (3 << 20, "ascending")):
        rng = np.random.default_rng(n)
        log = np.zeros(n, dtype=hetm.LOG_ENTRY)
        log["addr"] = rng.integers(0, W, n)
        log["value"] = rng.integers(0, 2**63, n, dtype=np.uint64)
        log["ts"] = (rng.permutation(n) if tsorder == "random" else np.arange(n)) + 1
        d = dev_factory(W, rs_gran_bytes=8, log_capacity=n)
        d.stream_chunk(log)
        assert not d.round_verdict()
        ts, want = np.zeros(W, np.uint64), np.zeros(W, np.uint64)
        orc.validate_chunk(log, np.zeros(W // 64, np.uint64), 8, ts, want)
        assert (d.download(hetm.REPLICA_DEV) == want).all(), tsorder
        # the queue is reset for the next launch: a second round on the same handle
        d.clear_round()
        log2 = log.copy()
        log2["ts"] += n
        log2["value"] ^= np.uint64(0x5555)
        d.stream_chunk(log2)
        assert not d.round_verdict()
        orc.validate_chunk(log2, np.zeros(W // 64, np.uint64), 8, ts, want)
        assert (d.download(hetm.REPLICA_DEV) == want).all(), tsorder


def test_validate_adaptive_apply_modes(hetm, orc, dev_factory):
    """The apply pass switches between its exchange form and its atomicMax form
    per launch, decided on the device from the duplicates the previous launch
    met (validate.cu apply_xchg_kernel): chunks alternating uniform and hot
    words, in both orders, with words repeating ACROSS launches of one round
    (an older entry arriving after a fresher one was applied), must leave the
    freshest value in every word after every chunk."""
    W = 1 << 13
    rng = np.random.default_rng(2024)
    d = dev_factory(W, rs_gran_bytes=8, log_capacity=1 << 16)
    ts, want = np.zeros(W, np.uint64), np.zeros(W, np.uint64)
    n = 1 << 14
    all_ts = rng.permutation(12 * n) + 1  # one round: ts unique, chunks arrive out of ts order
    for k, hot in enumerate([False, True, True, False, False, True, False, True, True, True, False, False]):
        log = np.zeros(n, dtype=hetm.LOG_ENTRY)
        log["addr"] = rng.integers(0, 64 if hot else W, n)
        log["value"] = rng.integers(0, 2**63, n, dtype=np.uint64)
        log["ts"] = all_ts[k * n:(k + 1) * n]
        d.stream_chunk(log, seq=k)
        assert not d.round_verdict()
        orc.validate_chunk(log, np.zeros(W // 64, np.uint64), 8, ts, want)
        assert (d.download(hetm.REPLICA_DEV) == want).all(), (k, hot)


def test_validate_permuted_delivery_orders(hetm, orc, dev_factory):
    """Acceptance #5 on the device: 10 delivery orders, same max-ts result."""
    W = 256
    rng = np.random.default_rng(99)
    log = random_log(rng, 4000, W)
    ts, want = np.zeros(W, np.uint64), np.zeros(W, np.uint64)
    orc.validate_chunk(log, np.zeros(4, np.uint64), 8, ts, want)
    chunks = np.array_split(log, 20)
    for rep in range(10):
        d = dev_factory(W, rs_gran_bytes=8)
        keep = [d.stream_chunk(chunks[k], seq=int(k)) for k in rng.permutation(20)]
        assert not d.round_verdict()
        assert (d.download(hetm.REPLICA_DEV) == want).all()
        del keep
        d.close()


@pytest.mark.parametrize("asynchronous", [False, True])
def test_false_positive_1k(hetm, orc, dev_factory, asynchronous):
    """device read word 0, host wrote word 127 -> conflict at 1 KiB;
    the clear (sync, or enqueued without a host sync) resets bitmaps and verdict."""
    d = dev_factory(1 << 17, rs_gran_bytes=1024)
    d.register_kernel(hetm.KERNEL_RW)
    d.execute_batch(hetm.KERNEL_RW, rw_txs(orc, [([0], [], [])]))
    log = np.array([(127, 1, 1)], dtype=hetm.LOG_ENTRY)
    d.stream_chunk(log)
    assert d.round_verdict()
    d.clear_round(asynchronous=asynchronous)
    d.sync()
    assert d.bitmap_stats() == (0, 0, 0)
    d.execute_batch(hetm.KERNEL_RW, rw_txs(orc, [([0], [], [])]))
    log2 = np.array([(128, 1, 2)], dtype=hetm.LOG_ENTRY)
    d.stream_chunk(log2)
    assert not d.round_verdict()


def test_validate_only_then_apply(hetm, orc, dev_factory):
    W = 1024
    d = dev_factory(W, rs_gran_bytes=8)
    rng = np.random.default_rng(1)
    log = random_log(rng, 3000, W)
    keep = [d.stream_chunk(c, mode=hetm.VALIDATE_ONLY) for c in np.array_split(log, 3)]
    assert not d.round_verdict()
    assert (d.download(hetm.REPLICA_DEV) == 0).all()  # validate-only: nothing applied
    d.apply_log()
    d.round_verdict()
    ts, want = np.zeros(W, np.uint64), np.zeros(W, np.uint64)
    orc.validate_chunk(log, np.zeros(16, np.uint64), 8, ts, want)
    assert (d.download(hetm.REPLICA_DEV) == want).all()
    del keep


def test_round_closed(hetm, dev_factory):
    d = dev_factory(64, rs_gran_bytes=8)
    d.close_intake()
    with pytest.raises(hetm.RoundClosedError):
        d.stream_chunk(np.array([(1, 1, 1)], dtype=hetm.LOG_ENTRY))
    d.open_intake()
    d.stream_chunk(np.array([(1, 1, 1)], dtype=hetm.LOG_ENTRY))
    d.round_verdict()


def test_empty_chunk_recorded(hetm, dev_factory):
    d = dev_factory(64, rs_gran_bytes=8)
    d.stream_chunk(np.zeros(0, hetm.LOG_ENTRY))  # SPEC.md:276 empty chunk delivery
    assert (hetm.H2D, hetm.TAG_LOG, 0) in d.transfer_log()


@pytest.mark.parametrize("asynchronous", [False, True])
def test_nonmonotone_ts_detected(hetm, dev_factory, asynchronous):
    d = dev_factory(64, rs_gran_bytes=8)
    d.stream_chunk(np.array([(1, 5, 100)], dtype=hetm.LOG_ENTRY))
    d.round_verdict()
    d.clear_round(asynchronous=asynchronous)  # the TS floor rolls to 100 either way
    d.stream_chunk(np.array([(2, 6, 50)], dtype=hetm.LOG_ENTRY))
    with pytest.raises(hetm.NonMonotoneTsError):
        d.round_verdict()
    d.clear_round(reset_ts=True, asynchronous=asynchronous)  # SPEC.md:421 literal reset; the flag clears
    d.stream_chunk(np.array([(2, 6, 50)], dtype=hetm.LOG_ENTRY))
    d.round_verdict()
    assert d.raw_read(hetm.REPLICA_DEV, 2) == 6


# ------------------------------------------------------------------ merge
def test_merge_commit_one_word_one_chunk(hetm, orc, dev_factory):
    """device wrote 1 word -> exactly 16384 bytes D2H."""
    W = 1 << 16
    d = dev_factory(W)
    d.register_kernel(hetm.KERNEL_RW)
    d.execute_batch(hetm.KERNEL_RW, rw_txs(orc, [([], [5000], [9])]))
    assert not d.round_verdict()
    d.clear_transfer_log()
    host = np.zeros(W, np.uint64)
    st = d.merge_commit(host)
    d.merge_wait()
    assert st.dirty_chunks == 1 and st.transfers == 1 and st.bytes_d2h == 16384
    assert [r for r in d.transfer_log() if r[0] == hetm.D2H] == [(hetm.D2H, hetm.TAG_MERGE, 16384)]
    assert host[5000] == 9
    assert (host == d.download(hetm.REPLICA_DEV)).all()
    assert (d.download(hetm.REPLICA_DEV_SHADOW) == host).all()


def test_merge_commit_coalescing(hetm, orc, dev_factory):
    """adjacent dirty chunks -> one record; separated -> two."""
    W = 1 << 16
    d = dev_factory(W)
    d.register_kernel(hetm.KERNEL_RW)
    d.execute_batch(hetm.KERNEL_RW, rw_txs(orc, [([], [0], [1]), ([], [2048], [1]), ([], [8192], [1])]))
    d.round_verdict()
    d.clear_transfer_log()
    host = np.zeros(W, np.uint64)
    d.merge_commit(host)
    d.merge_wait()
    assert [r[2] for r in d.transfer_log() if r[0] == hetm.D2H] == [32768, 16384]
    d.clear_round()
    d.clear_transfer_log()
    d.merge_commit(host)  # zero dirty chunks -> no D2H bytes
    d.merge_wait()
    assert [r for r in d.transfer_log() if r[0] == hetm.D2H] == []


def test_merge_commit_refuses_conflict(hetm, orc, dev_factory):
    d = dev_factory(1024, rs_gran_bytes=8)
    d.register_kernel(hetm.KERNEL_RW)
    d.execute_batch(hetm.KERNEL_RW, rw_txs(orc, [([3], [], [])]))
    d.stream_chunk(np.array([(3, 1, 1)], dtype=hetm.LOG_ENTRY))
    assert d.round_verdict()
    with pytest.raises(hetm.StateError):
        d.merge_commit(np.zeros(1024, np.uint64))


@pytest.mark.parametrize("optimized", [False, True])
def test_merge_abort_device_spec_378(hetm, orc, dev_factory, optimized):
    """Device wrote {3,9}; host wrote 3 (read by the device) -> dev[9] = round start,
    dev[3] = host value; devReplica == hostReplica."""
    W = 1 << 12
    d = dev_factory(W, rs_gran_bytes=8)
    d.register_kernel(hetm.KERNEL_RW)
    start = np.arange(W, dtype=np.uint64) * 3
    d.upload(hetm.REPLICA_DEV, 0, start)
    host = start.copy()
    d.merge_commit(host)  # establish shadow == round start
    d.merge_wait()
    d.clear_round()
    d.execute_batch(hetm.KERNEL_RW, rw_txs(orc, [([], [3], [100]), ([], [9], [100])]))
    host[3] = 777
    d.stream_chunk(np.array([(3, 777, 10)], dtype=hetm.LOG_ENTRY))
    assert d.round_verdict()
    d.merge_abort_device(host, optimized=optimized)
    got = d.download(hetm.REPLICA_DEV)
    assert got[9] == start[9] and got[3] == 777
    assert (got == host).all()
    assert (d.download(hetm.REPLICA_DEV_SHADOW) == host).all()


def test_merge_abort_basic_equals_optimized(hetm, orc, dev_factory):
    """Acceptance #6: paired seeds, basic and optimized rollback identical."""
    W = 1 << 16
    finals = []
    for optimized in (False, True):
        d = dev_factory(W, rs_gran_bytes=1024)
        d.register_kernel(hetm.KERNEL_BANK)
        init = np.full(W, 1000, np.uint64)
        d.upload(hetm.REPLICA_DEV, 0, init)
        host = init.copy()
        d.merge_commit(host)
        d.merge_wait()
        d.clear_round()
        txs = orc.gen_bank_batch(5, 20000, 0, W)
        d.execute_batch(hetm.KERNEL_BANK, txs)
        rng = np.random.default_rng(6)
        log = random_log(rng, 30000, W, ts0=0)
        orc.apply_log_ts_order(host, log)
        keep = [d.stream_chunk(c) for c in np.array_split(log, 7)]
        assert d.round_verdict()
        d.merge_abort_device(host, optimized=optimized)
        got = d.download(hetm.REPLICA_DEV)
        assert (got == host).all()
        finals.append(got)
        del keep
    assert (finals[0] == finals[1]).all()


def test_merge_abort_host_spec_387(hetm, orc, dev_factory):
    """FavorDevice: host wrote 2, device read 2 and wrote 4 -> 2 = round start, 4 = device value."""
    W = 1024
    d = dev_factory(W, rs_gran_bytes=8)
    d.register_kernel(hetm.KERNEL_RW)
    snap = np.arange(W, dtype=np.uint64)
    d.upload(hetm.REPLICA_DEV, 0, snap)
    host = snap.copy()
    d.merge_commit(host)
    d.merge_wait()
    d.clear_round()
    d.execute_batch(hetm.KERNEL_RW, rw_txs(orc, [([2], [4], [0])]))  # w4 = old4 + old2
    host[2] = 999
    d.stream_chunk(np.array([(2, 999, 1)], dtype=hetm.LOG_ENTRY), mode=hetm.VALIDATE_ONLY)
    assert d.round_verdict()
    d.merge_abort_host(host, snap)
    assert host[2] == snap[2] and host[4] == snap[4] + snap[2]
    assert (host == d.download(hetm.REPLICA_DEV)).all()


# --------------------------------------------------------- round sequences
@pytest.mark.parametrize("optimized", [False, True])
def test_rounds_match_sequential_replay(hetm, orc, dev_factory, optimized):
    """Acceptance #1/#2: per round, host txs in ts order then
    device txs in ticket order; replicas equal after every round; verdict ==
    bruteForceIntersect."""
    W, gran = 1 << 14, 1024
    rng = np.random.default_rng(12)
    d = dev_factory(W, rs_gran_bytes=gran)
    d.register_kernel(hetm.KERNEL_BANK)
    host = np.full(W, 100, np.uint64)
    d.upload(hetm.REPLICA_DEV, 0, host)
    d.merge_commit(host)
    d.merge_wait()
    d.clear_round()
    ref = host.copy()
    ts0 = 0
    outcomes = []
    for rnd in range(8):
        overlap = rnd % 3 == 2  # host writes into the device half every third round
        txs = orc.gen_bank_batch(rnd + 1, 4000, 0, W // 2)
        r = d.execute_batch(hetm.KERNEL_BANK, txs)
        lo = 0 if overlap else W // 2
        log = orc.gen_host_log(50 + rnd, 500, 2, 4, lo, W // 2, ts_base=ts0)
        ts0 += 500
        orc.apply_log_ts_order(host, log)  # the host's own replica
        keep = [d.stream_chunk(c, src_thread=i) for i, c in enumerate(np.array_split(log, 5))]
        conflict = d.round_verdict()
        order = orc.order_by_ticket(r.tickets)
        probe = np.zeros(W, np.uint64)
        rs_bits, _, _ = orc.bank_replay(probe, txs, order, gran, 16384)
        assert conflict == orc.brute_force_intersect(log, rs_bits, W * 8 // gran, gran)
        orc.apply_log_ts_order(ref, log)
        if conflict:
            d.merge_abort_device(host, optimized=optimized)
        else:
            orc.bank_replay(ref, txs, order, gran, 16384)
            d.merge_commit(host)
            d.merge_wait()
        d.clear_round()
        outcomes.append(conflict)
        assert (host == ref).all()
        assert (d.download(hetm.REPLICA_DEV) == host).all()
        del keep
    assert any(outcomes) and not all(outcomes)


@pytest.mark.parametrize("batches", [1, 3])
def test_merge_delta_rounds_match_replay(hetm, orc, dev_factory, batches):
    """mergeCommit in delta form (HETM_CFG_MERGE_DELTA): sparse device write
    sets ship as 12-B {word, value} records; the host replica must end exactly
    as with the SPEC chunk copy (replica equality after every round,
    SPEC.md:640), across several batches per round and aborted rounds."""
    W, gran = 1 << 20, 1024
    d = dev_factory(W, rs_gran_bytes=gran, merge_delta=True)
    d.register_kernel(hetm.KERNEL_BANK)
    host = np.full(W, 7, np.uint64)
    d.upload(hetm.REPLICA_DEV, 0, host)
    d.merge_commit(host)
    d.merge_wait()
    d.clear_round()
    ref = host.copy()
    ts0, outcomes = 0, []
    for rnd in range(6):
        overlap = rnd == 3
        tks, all_txs, n_tickets = [], [], 0
        for b in range(batches):
            txs = orc.gen_bank_batch(100 * rnd + b + 1, 3000, 0, W // 2)
            r = d.execute_batch(hetm.KERNEL_BANK, txs)
            tks.append(r.tickets)
            n_tickets += r.ticket_end - r.ticket_first  # includes tickets of aborted attempts
            all_txs.append(txs)
        txs = np.concatenate(all_txs)
        tickets = np.concatenate(tks)
        log = orc.gen_host_log(70 + rnd, 800, 2, 4, 0 if overlap else W // 2, W // 2, ts_base=ts0)
        ts0 += 800
        orc.apply_log_ts_order(host, log)
        keep = [d.stream_chunk(c, src_thread=i) for i, c in enumerate(np.array_split(log, 4))]
        conflict = d.round_verdict()
        orc.apply_log_ts_order(ref, log)
        d.clear_transfer_log()
        if conflict:
            d.merge_abort_device(host, optimized=True)
        else:
            orc.bank_replay(ref, txs, orc.order_by_ticket(tickets), gran, 16384)
            st = d.merge_commit(host)
            d.merge_wait()
            n_slots = 2 * n_tickets  # records: 8 B each by zero-copy stores, 12 B each by DMA
            recs = [t[2] for t in d.transfer_log() if t[:2] == (hetm.D2H, hetm.TAG_MERGE_DELTA)]
            assert st.bytes_d2h == sum(recs) and 8 * n_slots <= st.bytes_d2h <= 12 * n_slots
        d.clear_round()
        outcomes.append(conflict)
        assert (host == ref).all(), rnd
        assert (d.download(hetm.REPLICA_DEV) == host).all(), rnd
        assert (d.download(hetm.REPLICA_DEV_SHADOW) == host).all(), rnd
        del keep
    assert any(outcomes) and not all(outcomes)


def test_merge_delta_falls_back_to_chunks_when_dense(hetm, orc, dev_factory):
    """Dense write sets (more record bytes than dirty-chunk bytes) use the
    SPEC chunk copy even with HETM_CFG_MERGE_DELTA."""
    W = 1 << 14
    d = dev_factory(W, merge_delta=True)
    d.register_kernel(hetm.KERNEL_BANK)
    host = np.zeros(W, np.uint64)
    txs = orc.gen_bank_batch(3, 6000, 0, W // 2)
    r = d.execute_batch(hetm.KERNEL_BANK, txs)
    assert not d.round_verdict()
    d.clear_transfer_log()
    st = d.merge_commit(host)
    d.merge_wait()
    assert st.bytes_d2h == st.dirty_chunks * 16384
    assert all(t[1] == hetm.TAG_MERGE for t in d.transfer_log() if t[0] == hetm.D2H)
    ref = np.zeros(W, np.uint64)
    orc.bank_replay(ref, txs, orc.order_by_ticket(r.tickets), 1024, 16384)
    assert (host == ref).all()


# ------------------------------------------- cfg3: zipf hot spot (abort path)
@pytest.mark.parametrize("W,n,alpha", [(1 << 16, 1 << 14, 0.99), (1 << 20, 1 << 16, 0.99), (1 << 20, 1 << 15, 1.5)])
def test_cfg3_zipf_batch_replays(hetm, orc, dev_factory, W, n, alpha):
    """BASELINE configs[2] shape: zipf-skewed bank accounts (hot words contended
    by thousands of transactions of one batch): every transaction commits and
    the ticket-order replay reproduces the STMR and the bitmaps bit-exactly."""
    d = dev_factory(W, rs_gran_bytes=1024)
    d.register_kernel(hetm.KERNEL_BANK)
    init = np.full(W, 1000, np.uint64)
    d.upload(hetm.REPLICA_DEV, 0, init)
    txs = orc.gen_bank_batch(31, n, 0, W, zipf=alpha)
    r = d.execute_batch(hetm.KERNEL_BANK, txs)
    assert r.committed == n
    ref = check_replay(hetm, orc, d, txs, r.tickets, init, 1024, 16384)
    assert int(ref.sum(dtype=np.uint64)) == (1000 * W) % (1 << 64)


@pytest.mark.parametrize("optimized", [False, True])
def test_cfg3_zipf_rounds_roll_back(hetm, orc, dev_factory, optimized):
    """CPU and GPU draw from the same zipf hot set: the host log hits words the
    device read, every round is DeviceAborted and rolled back;
    the device replica must equal the host-only replay after every round."""
    W, gran = 1 << 20, 1024
    d = dev_factory(W, rs_gran_bytes=gran, merge_delta=True)
    d.register_kernel(hetm.KERNEL_BANK)
    host = np.full(W, 500, np.uint64)
    d.upload(hetm.REPLICA_DEV, 0, host)
    d.merge_commit(host)
    d.merge_wait()
    d.clear_round()
    ts0 = 0
    for rnd in range(4):
        txs = orc.gen_bank_batch(200 + rnd, 1 << 14, 0, W, zipf=0.99)
        r = d.execute_batch(hetm.KERNEL_BANK, txs)
        assert r.committed == txs.size
        log = orc.gen_host_log(300 + rnd, 4000, 2, 8, 0, W, ts_base=ts0, zipf=0.99)
        ts0 += 4000
        orc.apply_log_ts_order(host, log)
        keep = [d.stream_chunk(c, src_thread=i) for i, c in enumerate(np.array_split(log, 8))]
        assert d.round_verdict(), "zipf host log must hit the device read set"
        d.merge_abort_device(host, optimized=optimized)
        d.clear_round()
        assert (d.download(hetm.REPLICA_DEV) == host).all(), rnd
        del keep


@pytest.mark.slow
def test_cfg3_zipf_full_size(hetm, orc, dev_factory):
    """BASELINE configs[2] at size: 1 GiB STMR, 2^20 zipf(0.99) bank transactions,
    a 2^20-entry zipf host log on the same range -> conflict -> optimized
    rollback; replay parity, bank sum, and replica equality after the abort."""
    W, n = 1 << 27, 1 << 20
    d = dev_factory(W, rs_gran_bytes=1024)
    d.register_kernel(hetm.KERNEL_BANK)
    init = np.full(W, 1000, np.uint64)
    d.upload(hetm.REPLICA_DEV, 0, init)
    d.merge_commit(init)
    d.merge_wait()
    d.clear_round()
    txs = orc.gen_bank_batch(2025, n, 0, W, zipf=0.99)
    r = d.execute_batch(hetm.KERNEL_BANK, txs)
    assert r.committed == n
    ref = check_replay(hetm, orc, d, txs, r.tickets, init, 1024, 16384)
    assert int(ref.sum(dtype=np.uint64)) == (1000 * W) % (1 << 64)
    log = orc.gen_host_log(77, n // 2, 2, 8, 0, W, ts_base=0, zipf=0.99)
    host = init.copy()
    orc.apply_log_ts_order(host, log)
    keep = [d.stream_chunk(c, src_thread=i) for i, c in enumerate(np.array_split(log, 8))]
    assert d.round_verdict()
    d.merge_abort_device(host, optimized=True)
    assert (d.download(hetm.REPLICA_DEV) == host).all()
    del keep


# ------------------------------------ cfg4: MemcachedGPU-style cache GET/SET
def check_cache_replay(hetm, orc, d, txs, r, init, n_sets, gran=1024, chunk=16384):
    order = orc.order_by_ticket(r.tickets)
    assert order.size == txs.size
    ref = init.copy()
    res, rs, ws, ch = orc.cache_replay(ref, txs, r.tickets, n_sets, gran, chunk)
    got = d.download(hetm.REPLICA_DEV)
    assert (got == ref).all(), f"{int((got != ref).sum())} words differ from ticket-order replay"
    assert (r.results == res).all(), "GET/SET results differ"
    assert (d.snapshot(hetm.BMP_RS).words == rs).all()
    assert (d.snapshot(hetm.BMP_WS).words == ws).all()
    assert (d.snapshot(hetm.BMP_CHUNK).words == ch).all()
    assert ((ws & ~rs) == 0).all()
    return ref


@pytest.mark.parametrize("sched", ["optimistic", "scan"])
@pytest.mark.parametrize("gran", GRANS)
@pytest.mark.parametrize("n_sets,n,alpha", [(64, 1 << 12, 0.5), (1024, 1 << 14, 0.5), (1 << 14, 1 << 16, 0.99)])
def test_cache_batch_replays(hetm, orc, dev_factory, gran, n_sets, n, alpha, sched):
    """GET/SET 90/10 (BASELINE configs[3]) after a warm-up SET batch: STMR,
    per-transaction results and bitmaps equal the ticket-order replay, for the
    optimistic kernel and the set-sequential SCAN schedule (input order)."""
    W = n_sets * 64
    d = dev_factory(W, rs_gran_bytes=gran)
    d.register_kernel(hetm.KERNEL_CACHE)
    d.set_schedule(hetm.SCHED_SCAN if sched == "scan" else hetm.SCHED_OPTIMISTIC)
    init = np.zeros(W, np.uint64)
    warm = orc.gen_cache_batch(1, n, n_sets * 4, alpha, get_permille=0, part=-1, steal_permille=500)
    r = d.execute_batch(hetm.KERNEL_CACHE, warm, results=True)
    ref = check_cache_replay(hetm, orc, d, warm, r, init, n_sets, gran)
    d.clear_round()
    txs = orc.gen_cache_batch(2, n, n_sets * 4, alpha, get_permille=900, part=-1, steal_permille=500)
    r = d.execute_batch(hetm.KERNEL_CACHE, txs, results=True)
    check_cache_replay(hetm, orc, d, txs, r, ref, n_sets, gran)
    st = r.results["status"]
    assert (st == hetm.CACHE_HIT).any() and (st == hetm.CACHE_MISS).any()
    if sched == "scan":
        assert r.aborts == 0 and (r.tickets == r.ticket_first + np.arange(n, dtype=np.uint64)).all()


@pytest.mark.parametrize("sched", ["optimistic", "scan"])
@pytest.mark.parametrize("steal", [0, 1000])
def test_cache_rounds_against_host(hetm, orc, dev_factory, steal, sched):
    """routing by the key's last bit -> no inter-device
    conflict (steal 0); the GPU taking the CPU's keys (steal 1000) conflicts
    and rolls back.  Replicas equal after every round."""
    n_sets = 1 << 12
    W = n_sets * 64
    d = dev_factory(W, rs_gran_bytes=1024, merge_delta=True)
    d.register_kernel(hetm.KERNEL_CACHE)
    d.set_schedule(hetm.SCHED_SCAN if sched == "scan" else hetm.SCHED_OPTIMISTIC)
    host = np.zeros(W, np.uint64)
    outcomes = []
    ts = 0
    for rnd in range(4):
        gpu = orc.gen_cache_batch(10 + rnd, 1 << 13, 1 << 14, 0.5, 900 if rnd else 0, part=-1,
                                  steal_permille=steal)
        r = d.execute_batch(hetm.KERNEL_CACHE, gpu, results=True)
        cpu = orc.gen_cache_batch(20 + rnd, 1 << 11, 1 << 14, 0.5, 900 if rnd else 0, part=0)
        _, log = orc.cache_host_run(host, cpu, n_sets, ts_base=ts)
        ts += cpu.size
        keep = [d.stream_chunk(c, src_thread=i) for i, c in enumerate(np.array_split(log, 4))]
        conflict = d.round_verdict()
        if conflict:
            d.merge_abort_device(host, optimized=True)
        else:
            orc.cache_replay(host, gpu, r.tickets, n_sets, 1024, 16384)
            d.merge_commit(host)
            d.merge_wait()
        d.clear_round()
        outcomes.append(conflict)
        assert (d.download(hetm.REPLICA_DEV) == host).all(), rnd
        del keep
    if steal == 0:
        assert not any(outcomes)
    else:
        assert all(outcomes)


@pytest.mark.slow
def test_cfg4_cache_full_size(hetm, orc, dev_factory):
    """BASELINE configs[3] geometry: 2^20 sets x 8 ways (512 MiB of words),
    a 2^20-transaction SET warm-up then a 2^20 GET/SET 90/10 batch (zipf 0.5)."""
    n_sets, n = 1 << 20, 1 << 20
    W = n_sets * 64
    d = dev_factory(W, rs_gran_bytes=1024)
    d.register_kernel(hetm.KERNEL_CACHE)
    init = np.zeros(W, np.uint64)
    warm = orc.gen_cache_batch(7, n, 1 << 22, 0.5, get_permille=0, part=1)
    r = d.execute_batch(hetm.KERNEL_CACHE, warm, results=True)
    ref = check_cache_replay(hetm, orc, d, warm, r, init, n_sets)
    d.clear_round()
    txs = orc.gen_cache_batch(8, n, 1 << 22, 0.5, get_permille=900, part=1)
    r = d.execute_batch(hetm.KERNEL_CACHE, txs, results=True)
    check_cache_replay(hetm, orc, d, txs, r, ref, n_sets)


# ------------------------------------------------------------ shard router
@pytest.mark.parametrize("n,G", [(100003, 8), (5, 3), (70001, 40), (1 << 20, 64), (4097, 1)])
def test_route_log_partitions_stably(hetm, dev_factory, n, G):
    torch = pytest.importorskip("torch")
    d = dev_factory(1024)
    rng = np.random.default_rng(n + G)
    sw = 1 << 20
    log = random_log(rng, n, G * sw)
    src = torch.from_numpy(log.view(np.uint64).reshape(-1).astype(np.int64)).cuda()
    dst = torch.empty_like(src)
    counts = torch.zeros(G, dtype=torch.int64, device="cuda")
    d.route_log_dptr(src.data_ptr(), n, G, sw, dst.data_ptr(), counts.data_ptr())
    torch.cuda.synchronize()
    d.sync()
    out = dst.cpu().numpy().view(np.uint64).view(hetm.LOG_ENTRY)
    owner = log["addr"] // sw
    want = np.concatenate([log[owner == s] for s in range(G)])
    assert counts.cpu().tolist() == [int((owner == s).sum()) for s in range(G)]
    assert out.tobytes() == want.tobytes()


# -------------------------------------------------- BASELINE-size properties
@pytest.mark.slow
def test_cfg2_bank_full_size(hetm, orc, dev_factory):
    """BASELINE configs[1]: 1 GiB STMR (2^27 words), one 2^20-tx batch; replay in
    ticket order reproduces the STMR bit-exactly and preserves the bank sum."""
    W, n = 1 << 27, 1 << 20
    d = dev_factory(W, rs_gran_bytes=1024)
    d.register_kernel(hetm.KERNEL_BANK)
    init = np.full(W, 1000, np.uint64)
    d.upload(hetm.REPLICA_DEV, 0, init)
    txs = orc.gen_bank_batch(2024, n, 0, W // 2)
    r = d.execute_batch(hetm.KERNEL_BANK, txs)
    assert r.committed == n
    ref = check_replay(hetm, orc, d, txs, r.tickets, init, 1024, 16384)
    assert int(ref.sum(dtype=np.uint64)) == (1000 * W) % (1 << 64)


@pytest.mark.slow
def test_cfg5_validate_full_shard(hetm, orc, dev_factory):
    """Validation+apply on a 1 GiB shard with a 4M-entry duplicate-heavy log."""
    W, n = 1 << 27, 1 << 22
    rng = np.random.default_rng(5)
    d = dev_factory(W, rs_gran_bytes=1024, shadow=False)
    nbits = W * 8 // 1024
    rs = np.zeros(nbits // 64, np.uint64)
    hot = rng.choice(nbits, nbits // 1000, replace=False)
    np.bitwise_or.at(rs, hot >> 6, (np.uint64(1) << (hot & 63).astype(np.uint64)))
    d.or_bitmap(hetm.BMP_RS, rs)
    log = random_log(rng, n, W)
    log["addr"][: n // 10] = rng.integers(0, 1 << 16, n // 10)  # 10% from a 2^16-word hot set
    keep = [d.stream_chunk(c) for c in np.array_split(log, 8)]
    conflict = d.round_verdict()
    ts, dev = np.zeros(W, np.uint64), np.zeros(W, np.uint64)
    assert conflict == orc.validate_chunk(log, rs, 1024, ts, dev)
    assert (d.download(hetm.REPLICA_DEV) == dev).all()
    del keep
