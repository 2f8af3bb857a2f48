"""Device half of mergeCommit without a host round trip (hetm_dev_merge_stage,
SPEC.md:363-371) and the hand-written delta kernels (claim + emit, no sort):
committed rounds land bit-exactly in the host replica and devShadow; on a
conflict the staged kernels do nothing and the optimized rollback
 is still exact; entries validated from device memory are
retained in the round arena (HETM_RETAIN) or read from the peer receive
arena, so the shadow refresh stays incremental.  Checked against the oracle."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

W = 1 << 16
GRAN = 1024


def _bank_round(hetm, orc, d, torch, seed, host_lo, conflict_word=None, ts_base=0, retain=True):
    """One device-resident round: bank batch on [0, W/2), host log on
    [W/2, W) (+ one entry on `conflict_word`), validate_dptr APPLY, merge_stage."""
    B = 1 << 13
    txs = hetm.gen_bank_batch(seed, B, 0, W // 2)
    t_tx = torch.from_numpy(txs.view(np.uint8)).cuda()
    tk = torch.empty(B, dtype=torch.int64, device="cuda")
    d.execute_batch_dptr(hetm.KERNEL_BANK, t_tx.data_ptr(), B, tk.data_ptr())
    log = hetm.gen_host_log(seed + 1, 2048, 2, 8, host_lo, W // 2, ts_base=ts_base)
    if conflict_word is not None:
        log[-1]["addr"] = conflict_word
    t_log = torch.from_numpy(log.view(np.uint64).reshape(-1, 3).astype(np.int64)).cuda()
    d.validate_dptr(t_log.data_ptr(), log.size, hetm.APPLY | (hetm.RETAIN if retain else 0))
    d.merge_stage()
    return txs, tk, log, (t_tx, t_log)


@pytest.mark.parametrize("retain", [True, False])
def test_stage_then_commit_matches_oracle(hetm, orc, retain):
    torch = pytest.importorskip("torch")
    with hetm.GpuDevice(W, rs_gran_bytes=GRAN, merge_delta=True) as d:
        d.register_kernel(hetm.KERNEL_BANK)
        init = np.full(W, 1000, np.uint64)
        d.upload(hetm.REPLICA_DEV, 0, init)
        host = hetm.PinnedArray((W,), np.uint64)
        host.array[:] = init
        d.merge_commit(host.array)
        d.merge_wait()
        d.clear_round()
        ref = init.copy()
        for r in range(3):
            txs, tk, log, keep = _bank_round(hetm, orc, d, torch, 10 + r, W // 2, ts_base=r * 10_000, retain=retain)
            assert not d.round_verdict()
            ms = d.merge_commit(host.array)
            d.merge_wait()
            # oracle: host log (ts order) then the device batch in ticket order
            orc.apply_log_ts_order(ref, log)
            orc.bank_replay(ref, txs, orc.order_by_ticket(tk.cpu().numpy().view(np.uint64)), GRAN, 16384)
            host.array[W // 2:] = ref[W // 2:]  # the host replica holds the host's own commits
            assert (d.download(hetm.REPLICA_DEV) == ref).all(), r
            assert (d.download(hetm.REPLICA_DEV_SHADOW) == ref).all(), r
            assert (host.array == ref).all(), r
            assert ms.bytes_d2h > 0
            d.clear_round()
            del keep
        host.free()


def test_stage_on_conflict_leaves_shadow_for_rollback(hetm, orc):
    torch = pytest.importorskip("torch")
    with hetm.GpuDevice(W, rs_gran_bytes=GRAN, merge_delta=True) as d:
        d.register_kernel(hetm.KERNEL_BANK)
        init = np.full(W, 1000, np.uint64)
        d.upload(hetm.REPLICA_DEV, 0, init)
        host = hetm.PinnedArray((W,), np.uint64)
        host.array[:] = init
        d.merge_commit(host.array)
        d.merge_wait()
        d.clear_round()
        txs, tk, log, keep = _bank_round(hetm, orc, d, torch, 77, W // 2, conflict_word=5)
        # a device-read word written by the host: the round conflicts, the staged kernels did nothing
        assert (d.download(hetm.REPLICA_DEV_SHADOW) == init).all()
        assert d.round_verdict()
        with pytest.raises(hetm.HetmError):  # the round's execution is over
            d.execute_batch_dptr(hetm.KERNEL_BANK, keep[0].data_ptr(), 16, tk.data_ptr())
        d.merge_abort_device(None, True)
        ref = init.copy()
        orc.apply_log_ts_order(ref, log)
        assert (d.download(hetm.REPLICA_DEV) == ref).all()
        assert (d.download(hetm.REPLICA_DEV_SHADOW) == ref).all()
        host.free()


def test_delta_records_unique_and_grouped(hetm, orc):
    """Hot accounts (zipf): many write-set slots per word; the delta keeps one
    record per word (merge_prepare's speculative swap/undo relies on it) and
    the host replica after commit equals the oracle."""
    torch = pytest.importorskip("torch")
    with hetm.GpuDevice(W, rs_gran_bytes=GRAN, merge_delta=True) as d:
        d.register_kernel(hetm.KERNEL_BANK)
        init = np.full(W, 1000, np.uint64)
        d.upload(hetm.REPLICA_DEV, 0, init)
        host = hetm.PinnedArray((W,), np.uint64)
        host.array[:] = init
        d.merge_commit(host.array)
        d.merge_wait()
        d.clear_round()
        B = 1 << 14
        txs = hetm.gen_bank_batch(5, B, 0, W // 2, zipf=0.99)
        r = d.execute_batch(hetm.KERNEL_BANK, txs)
        assert not d.round_verdict()
        d.merge_prepare(host.array)  # speculative swap: undone and redone below
        d.merge_abort_device(None, True)   # undo path over the unique records
        assert (host.array == init).all()
        d.clear_round()
        r = d.execute_batch(hetm.KERNEL_BANK, txs)
        assert not d.round_verdict()
        d.merge_prepare(host.array)
        ms = d.merge_commit(host.array)
        d.merge_wait()
        ref = init.copy()
        orc.bank_replay(ref, txs, orc.order_by_ticket(r.tickets), GRAN, 16384)  # the aborted round left no trace
        assert (host.array == ref).all() and (d.download(hetm.REPLICA_DEV) == ref).all()
        written = np.unique(np.concatenate([txs["acct"][:, 0], txs["acct"][:, 1]]))
        assert ms.bytes_d2h == 12 * written.size  # one 12-B record per written word
        host.free()


def test_received_regions_keep_the_shadow_incremental(hetm, orc):
    """apply_received (the multi-GPU exchange) no longer forces a full shadow
    copy: the shadow patch and the optimized rollback read the receive arena."""
    torch = pytest.importorskip("torch")
    G, Ws, cap = 2, W // 2, 8192
    devs = [hetm.GpuDevice(Ws, shard_base=s * Ws, rs_gran_bytes=GRAN, merge_delta=True) for s in range(G)]
    arenas = [d.recv_arena(G, cap) for d in devs]
    ent, cnt = [a[0] for a in arenas], [a[1] for a in arenas]
    ts_all, want = np.zeros(G * Ws, np.uint64), np.zeros(G * Ws, np.uint64)
    logs = [orc.gen_host_log(3 + s, 2000, 2, 4, 0, G * Ws, ts_base=s * 4000) for s in range(G)]
    keep = []
    for s, d in enumerate(devs):
        t = torch.from_numpy(logs[s].view(np.uint64).reshape(-1, 3).astype(np.int64)).cuda()
        keep.append(t)
        d.route_to_peers_dptr(t.data_ptr(), t.shape[0], G, Ws, s, cap, 0, ent, cnt)
    for d in devs:
        d.sync()
    for d in devs:
        d.apply_received(0, hetm.APPLY)
    orc.validate_chunk(np.concatenate(logs), np.zeros(G * Ws * 8 // GRAN // 64, np.uint64), GRAN, ts_all, want)
    for s, d in enumerate(devs):
        assert not d.round_verdict()
        if s == 0:  # commit: the shadow patch reads the received regions
            host = np.zeros(Ws, np.uint64)
            d.merge_commit(host)
            d.merge_wait()
            assert (d.download(hetm.REPLICA_DEV_SHADOW, s * Ws, Ws) == want[:Ws]).all()
        else:  # optimized rollback re-applies the received regions
            d.merge_abort_device(None, True)
            assert (d.download(hetm.REPLICA_DEV, s * Ws, Ws) == want[Ws:]).all()
            assert (d.download(hetm.REPLICA_DEV_SHADOW, s * Ws, Ws) == want[Ws:]).all()
    for d in devs:
        d.close()
