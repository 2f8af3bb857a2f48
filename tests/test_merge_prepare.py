"""hetm_dev_merge_prepare: the delta merge staged right after the execution
phase (and, with the host replica, applied to it speculatively) must leave
exactly the state of the plain merge on commit, and exactly the pre-round host
replica on every abort path (replica equality)."""
import numpy as np
import pytest

from test_gpu_parity import dev_factory  # noqa: F401  (fixture)

pytestmark = pytest.mark.gpu

W = 1 << 18


def fresh(hetm, dev_factory, sched=None):
    d = dev_factory(W, rs_gran_bytes=1024, merge_delta=True)
    d.register_kernel(hetm.KERNEL_BANK)
    if sched is not None:
        d.set_schedule(sched)
    host = np.full(W, 1000, np.uint64)
    d.upload(hetm.REPLICA_DEV, 0, host)
    d.merge_commit(host)
    d.merge_wait()
    d.clear_round()
    return d, host


def stream(d, log):
    return [d.stream_chunk(c, src_thread=i) for i, c in enumerate(np.array_split(log, 4))]


@pytest.mark.parametrize("speculative", [True, False])
@pytest.mark.parametrize("zipf", [0.0, 0.99])
def test_prepared_commit_rounds(hetm, orc, dev_factory, speculative, zipf):
    d, host = fresh(hetm, dev_factory)
    ref = host.copy()
    ts = 0
    for rnd in range(4):
        txs = orc.gen_bank_batch(10 + rnd, 1 << 14, 0, W // 2, zipf=zipf)   # device half
        r = d.execute_batch(hetm.KERNEL_BANK, txs)
        orc.bank_replay(ref, txs, orc.order_by_ticket(r.tickets), 1024, 16384)
        log = orc.gen_host_log(20 + rnd, 2000, 2, 4, W // 2, W // 2, ts_base=ts)  # host half: no conflict
        ts += 2000
        orc.apply_log_ts_order(host, log)   # the host STM's own writes, during the execution phase
        orc.apply_log_ts_order(ref, log)
        d.merge_prepare(host if speculative else None)  # after the host cut-off
        keep = stream(d, log)
        assert not d.round_verdict()
        d.merge_commit(host)
        d.merge_wait()
        d.clear_round()
        assert (host == ref).all(), rnd
        assert (d.download(hetm.REPLICA_DEV) == ref).all(), rnd
        del keep


@pytest.mark.parametrize("optimized", [True, False])
def test_prepared_then_device_abort_restores_host(hetm, orc, dev_factory, optimized):
    """Zipf batches (a word written by many transactions: one record per word) then a
    conflicting host log: the speculative writes are undone, the host keeps its own."""
    d, host = fresh(hetm, dev_factory)
    ts = 0
    for rnd in range(3):
        txs = orc.gen_bank_batch(40 + rnd, 1 << 14, 0, W, zipf=0.99)
        d.execute_batch(hetm.KERNEL_BANK, txs)
        log = orc.gen_host_log(50 + rnd, 3000, 2, 4, 0, W, ts_base=ts, zipf=0.99)
        ts += 3000
        orc.apply_log_ts_order(host, log)  # the host STM's own writes, during the execution phase
        before = host.copy()
        d.merge_prepare(host)
        d.merge_wait()
        assert (host != before).any()  # the speculative merge did land
        keep = stream(d, log)
        assert d.round_verdict()
        d.merge_abort_device(host, optimized=optimized)  # undoes the speculation first
        d.clear_round()
        assert (host == before).all(), rnd
        assert (d.download(hetm.REPLICA_DEV) == host).all(), rnd
        del keep


def test_prepared_then_new_batch_is_restaged(hetm, orc, dev_factory):
    d, host = fresh(hetm, dev_factory)
    ref = host.copy()
    for k in range(2):
        txs = orc.gen_bank_batch(60 + k, 1 << 13, 0, W // 2)
        r = d.execute_batch(hetm.KERNEL_BANK, txs)
        orc.bank_replay(ref, txs, orc.order_by_ticket(r.tickets), 1024, 16384)
        d.merge_prepare(host)   # the second batch cancels (undoes) the first staging
    assert not d.round_verdict()
    d.merge_commit(host)
    d.merge_wait()
    assert (host == ref).all() and (d.download(hetm.REPLICA_DEV) == ref).all()


def test_prepared_then_host_abort(hetm, orc, dev_factory):
    """FavorDevice: HostAborted -> host replica = round-start snapshot + the device's writes."""
    d, host = fresh(hetm, dev_factory)
    snapshot = host.copy()
    txs = orc.gen_bank_batch(70, 1 << 14, 0, W, zipf=0.99)
    r = d.execute_batch(hetm.KERNEL_BANK, txs)
    ref = snapshot.copy()
    orc.bank_replay(ref, txs, orc.order_by_ticket(r.tickets), 1024, 16384)
    log = orc.gen_host_log(71, 3000, 2, 4, 0, W, ts_base=0, zipf=0.99)
    orc.apply_log_ts_order(host, log)  # the host's speculative round (to be discarded)
    d.merge_prepare(host)
    keep = [d.stream_chunk(c, src_thread=i, mode=hetm.VALIDATE_ONLY) for i, c in enumerate(np.array_split(log, 4))]
    assert d.round_verdict()
    d.merge_abort_host(host, snapshot)
    d.merge_wait()
    d.clear_round()
    assert (host == ref).all() and (d.download(hetm.REPLICA_DEV) == ref).all()
    del keep


def test_clear_without_merge_undoes_speculation(hetm, orc, dev_factory):
    d, host = fresh(hetm, dev_factory)
    before = host.copy()
    d.execute_batch(hetm.KERNEL_BANK, orc.gen_bank_batch(80, 1 << 12, 0, W))
    d.merge_prepare(host)
    d.merge_wait()
    d.clear_round()
    assert (host == before).all()


def test_prepare_is_a_noop_without_delta_merge(hetm, orc, dev_factory):
    d = dev_factory(W, rs_gran_bytes=1024)  # chunk merge
    d.register_kernel(hetm.KERNEL_BANK)
    host = np.full(W, 1000, np.uint64)
    d.upload(hetm.REPLICA_DEV, 0, host)
    txs = orc.gen_bank_batch(90, 1 << 12, 0, W)
    d.execute_batch(hetm.KERNEL_BANK, txs)
    before = host.copy()
    d.merge_prepare(host)
    d.merge_wait()
    assert (host == before).all()
    assert not d.round_verdict()
    d.merge_commit(host)
    d.merge_wait()
    assert (host == d.download(hetm.REPLICA_DEV)).all()


def test_prepared_for_another_replica(hetm, orc, dev_factory):
    """merge_prepare(A) speculatively, then merge_commit(B): A is put back, B gets the merge."""
    d, host_a = fresh(hetm, dev_factory)
    host_b = host_a.copy()
    ref = host_a.copy()
    txs = orc.gen_bank_batch(95, 1 << 13, 0, W)
    r = d.execute_batch(hetm.KERNEL_BANK, txs)
    orc.bank_replay(ref, txs, orc.order_by_ticket(r.tickets), 1024, 16384)
    before_a = host_a.copy()
    d.merge_prepare(host_a)
    assert not d.round_verdict()
    d.merge_commit(host_b)
    d.merge_wait()
    assert (host_a == before_a).all()
    assert (host_b == ref).all() and (d.download(hetm.REPLICA_DEV) == ref).all()
