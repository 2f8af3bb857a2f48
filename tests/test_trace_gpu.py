"""Checker traces of live engine rounds on the GPU.

build/trace_test runs FavorHost rounds (HostStm workers + bank batches,
partitions swapped every round, a conflicting round every third) with
tracing on and checks P1 / P2-dagger with the oracle's checker.  With no
fault both pass; each seeded mutation of the protocol (skip RS
test, skip TS freshness, skip rollback of a chunk, report device commits
before validation, drop a log chunk) must be caught.
"""
import json
import os
import subprocess

import numpy as np
import pytest

import oracle as O

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
EXE = os.path.join(ROOT, "build", "trace_test")

FAULT_SKIP_RS, FAULT_SKIP_TS, FAULT_SKIP_ROLLBACK = 1, 2, 4          # capi.h HETM_FAULT_*
ENGINE_EARLY_DEVICE_COMMIT, ENGINE_DROP_CHUNK = 1, 2                  # engine.hpp ENGINE_FAULT_*


def run(rounds, dev_fault=0, eng_fault=0, dump="", policy="host"):
    if not os.path.exists(EXE):
        pytest.skip("build/trace_test not built")
    out = subprocess.run([EXE, str(rounds), str(dev_fault), str(eng_fault), dump or "", policy], capture_output=True,
                         text=True, timeout=600)
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert lines, out.stdout + out.stderr
    return out.returncode, json.loads(lines[-1])


@pytest.mark.gpu
def test_live_rounds_pass_p1_and_p2dagger(tmp_path):
    path = str(tmp_path / "rounds.hetmtrace")
    rc, r = run(9, dump=path)
    assert rc == 0 and r["ok"] == 1, r
    assert r["p1"]["verdict"] == 0 and r["p2dagger"]["verdict"] == 0
    assert r["conflict_rounds"] == 3                     # rounds 2, 5, 8 conflict -> DeviceAborted
    assert r["p1"]["txs"] > 9 * 4096 * 0.6 and r["p2dagger"]["txs"] >= 3 * 4000
    # the dump parses in Python and re-checks identically
    header, ev = O.load_trace(path)
    assert header["sizeWords"] == 1 << 18 and len(ev) == r["events"]
    init = np.full(header["sizeWords"], 1000, np.uint64)
    p1 = O.check_p1(ev, init)
    assert p1.verdict == O.CHECK_PASS and p1.checked_reads == r["p1"]["reads"]
    assert O.check_p2dagger(ev, init).verdict == O.CHECK_PASS


@pytest.mark.gpu
def test_live_rounds_favor_device_pass():
    """FavorDevice: the conflicting rounds are HostAborted — P2-dagger then checks the
    host transactions' speculative set (on the round-start state), P1 the rest."""
    rc, r = run(9, policy="device")
    assert rc == 0 and r["ok"] == 1 and r["policy"] == "FavorDevice", r
    assert r["conflict_rounds"] == 3 and r["p2dagger"]["txs"] > 0


@pytest.mark.gpu
@pytest.mark.parametrize("dev_fault,eng_fault,name", [
    (FAULT_SKIP_RS, 0, "skip RS test"),
    (FAULT_SKIP_TS, 0, "skip TS freshness"),
    (FAULT_SKIP_ROLLBACK, 0, "skip rollback of a chunk"),
    (0, ENGINE_EARLY_DEVICE_COMMIT, "report device commits before validation"),
    (0, ENGINE_DROP_CHUNK, "drop a log chunk"),
])
def test_mutations_are_caught(dev_fault, eng_fault, name):
    rc, r = run(9, dev_fault, eng_fault)
    assert rc == 0 and r["ok"] == 1, (name, r)
    assert r["p1"]["verdict"] == O.CHECK_FAIL or r["p2dagger"]["verdict"] == O.CHECK_FAIL


def _replay_records(state, txs, rec, kernel):
    """Ticket-order replay: every recorded read equals the serial state, every recorded write
    is what the transaction computes (bank: acct0 -= amount, acct1 += amount; rw: add + sum)."""
    committed = np.nonzero(rec[:, 0] != np.uint64(2**64 - 1))[0]
    order = committed[np.argsort(rec[committed, 0], kind="stable")]
    for i in order:
        r = rec[i]
        if kernel == "bank":
            a = [int(x) for x in txs["acct"][i]]
            assert [int(state[x]) for x in a] == [int(v) for v in r[1:5]], i
            assert int(r[7]) == (int(state[a[0]]) - int(txs["amount"][i])) % 2**64
            assert int(r[8]) == (int(state[a[1]]) + int(txs["amount"][i])) % 2**64
            state[a[0]], state[a[1]] = r[7], r[8]
        else:
            t = txs[i]
            s = 0
            for j in range(int(t["nr"])):
                assert int(state[t["r_addr"][j]]) == int(r[1 + j]), i
                s += int(r[1 + j])
            for j in range(int(t["nw"])):
                w = int(t["w_addr"][j])
                assert int(state[w]) == int(r[5 + j]), i
                assert int(r[7 + j]) == (int(r[5 + j]) + int(t["add"][j]) + s) % 2**64
                state[w] = r[7 + j]
    return len(order)


@pytest.mark.gpu
@pytest.mark.parametrize("sched", ["optimistic", "scan"])
@pytest.mark.parametrize("hot", [False, True])
def test_device_trace_records_match_ticket_replay(hot, sched):
    """hetm_dev_trace_next_batch: the traced bank batch's per-transaction read / write values are
    exactly what the ticket-order serial replay reads and writes (hot = contended 256-account span),
    for both schedules."""
    import paper_1905_00661_b200 as hetm
    W, B = 1 << 16, 1 << 13
    d = hetm.GpuDevice(W, rs_gran_bytes=1024)
    d.register_kernel(hetm.KERNEL_BANK)
    d.set_schedule(hetm.SCHED_SCAN if sched == "scan" else hetm.SCHED_OPTIMISTIC)
    init = (np.arange(W, dtype=np.uint64) * np.uint64(7919)) % np.uint64(100000)
    d.upload(hetm.REPLICA_DEV, 0, init)
    txs = hetm.gen_bank_batch(11, B, 0, 256 if hot else W)
    rec = np.zeros(B * hetm.TRACE_TX_WORDS, np.uint64)
    d.trace_next_batch(rec)
    r = d.execute_batch(hetm.KERNEL_BANK, txs)
    rec = rec.reshape(B, hetm.TRACE_TX_WORDS)
    assert (rec[:, 0] == r.tickets).all()
    state = init.copy()
    assert _replay_records(state, txs, rec, "bank") == r.committed == B
    assert (d.download(hetm.REPLICA_DEV, 0, W) == state).all()
    # the next (untraced) batch leaves the buffer alone
    rec2 = rec.copy()
    d.execute_batch(hetm.KERNEL_BANK, hetm.gen_bank_batch(12, 64, 0, W))
    assert (rec == rec2).all()


@pytest.mark.gpu
def test_device_trace_records_rw_kernel():
    import paper_1905_00661_b200 as hetm
    W, B = 1 << 12, 1 << 12
    d = hetm.GpuDevice(W, rs_gran_bytes=8)
    d.register_kernel(hetm.KERNEL_RW)
    rng = np.random.default_rng(3)
    txs = np.zeros(B, hetm.RW_TX)
    txs["nr"] = rng.integers(0, 5, B)
    txs["nw"] = rng.integers(1, 3, B)
    txs["r_addr"] = rng.integers(0, W, (B, 4))
    w = rng.integers(0, W, (B, 2))
    w[:, 1] = np.where(w[:, 1] == w[:, 0], (w[:, 0] + 1) % W, w[:, 1])  # distinct RMW words
    txs["w_addr"] = w
    txs["add"] = rng.integers(1, 100, (B, 2))
    rec = np.zeros(B * hetm.TRACE_TX_WORDS, np.uint64)
    d.trace_next_batch(rec)
    r = d.execute_batch(hetm.KERNEL_RW, txs)
    rec = rec.reshape(B, hetm.TRACE_TX_WORDS)
    state = np.zeros(W, np.uint64)
    assert _replay_records(state, txs, rec, "rw") == r.committed == B
    assert (d.download(hetm.REPLICA_DEV, 0, W) == state).all()
