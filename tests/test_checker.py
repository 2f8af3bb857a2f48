"""P1 / P2-dagger checker on hand-built traces (CPU).

The GPU-side end-to-end use — traces of live engine rounds, and the mutation
suite the checker must reject — is tests/test_trace_gpu.py.
"""
import os
import subprocess

import numpy as np
import pytest

import oracle as O

HOST, DEV = 0, 1
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


class TB:
    """Builds a trace in seq order, like the engine's recorder."""

    def __init__(self):
        self.ev = []
        self.round = 0

    def add(self, dev, kind, tx, addr=0, value=0):
        self.ev.append((len(self.ev), tx, addr, value, self.round, dev, kind, 0))

    def begin_round(self, r):
        self.round = r
        self.add(HOST, O.EV_ROUND, 0, 0, r)

    def tx(self, dev, tx, ops, commit_key, final=True):
        """ops: [("r"|"w", addr, value)], then SPEC_COMMIT(commit_key) and, at once, the round verdict."""
        self.add(dev, O.EV_BEGIN, tx)
        for op, a, v in ops:
            self.add(dev, O.EV_READ if op == "r" else O.EV_WRITE, tx, a, v)
        self.add(dev, O.EV_SPEC_COMMIT, tx, 0, commit_key)
        if final is not None:
            self.verdict(dev, tx, final)

    def verdict(self, dev, tx, final):
        self.add(dev, O.EV_FINAL_COMMIT if final else O.EV_ABORT, tx, 0,
                 self.round if final else O.ABORT_ROUND)

    def events(self):
        return np.array(self.ev, dtype=O.TRACE_EVENT)


D = 1 << 63  # device tx id bit


def test_empty_trace_passes():
    init = np.zeros(8, np.uint64)
    assert O.check_p1(np.zeros(0, O.TRACE_EVENT), init).verdict == O.CHECK_PASS
    assert O.check_p2dagger(np.zeros(0, O.TRACE_EVENT), init).verdict == O.CHECK_PASS


def committed_round_trace():
    """Round 0: host T1 (ts 1) x0 += 5; device D0 (ticket 0) x1 += 1 reading x2; host-then-device order."""
    t = TB()
    t.begin_round(0)
    t.tx(HOST, 1, [("r", 0, 10), ("w", 0, 15)], 1)
    t.tx(DEV, D | 0, [("r", 1, 20), ("r", 2, 30), ("w", 1, 21)], 0)
    t.begin_round(1)  # round 1: the device reads the host's round-0 write, the host the device's
    t.tx(DEV, D | 1 << 32, [("r", 0, 15), ("w", 0, 16)], 1)
    t.tx(HOST, 2, [("r", 1, 21)], 1)  # read-only at rv = 1
    return t


def test_committed_rounds_pass_with_counts():
    init = np.array([10, 20, 30, 0], np.uint64)
    r = O.check_p1(committed_round_trace().events(), init)
    assert r.verdict == O.CHECK_PASS, (r.reason, r.tx, r.addr, r.expected, r.got)
    assert r.checked_txs == 4 and r.checked_reads == 5


def test_inconsistent_read_fails_with_witness():
    """The device read x0 before the host's same-round write: host-then-device order cannot explain it
    (what a deleted RS test lets through)."""
    t = TB()
    t.begin_round(0)
    t.tx(HOST, 1, [("r", 0, 10), ("w", 0, 15)], 1)
    t.tx(DEV, D | 0, [("r", 0, 10), ("w", 0, 11)], 0)
    init = np.array([10, 0], np.uint64)
    r = O.check_p1(t.events(), init)
    assert r.verdict == O.CHECK_FAIL and r.reason == O.REASON_READ
    assert (r.tx, r.addr, r.expected, r.got, r.round) == (D | 0, 0, 15, 10, 0)


def test_host_observing_device_speculation_fails():
    """a host tx observing a device spec-committed (never finally committed) value -> fail."""
    t = TB()
    t.begin_round(0)
    t.tx(HOST, 1, [("r", 3, 0), ("w", 3, 1)], 1)
    t.tx(DEV, D | 0, [("r", 0, 10), ("w", 0, 99)], 0, final=False)  # DeviceAborted round
    t.begin_round(1)
    t.tx(HOST, 2, [("r", 0, 99)], 1)  # sees the rolled-back device write
    init = np.array([10, 0, 0, 0], np.uint64)
    r = O.check_p1(t.events(), init)
    assert r.verdict == O.CHECK_FAIL and r.reason == O.REASON_READ and r.tx == 2 and r.expected == 10
    assert O.check_p2dagger(t.events(), init).verdict == O.CHECK_PASS  # the device's own speculation is fine


def test_same_device_speculation_passes_p2dagger():
    """a device tx reading another device tx's spec-committed write, round later aborted."""
    t = TB()
    t.begin_round(0)
    t.tx(DEV, D | 0, [("r", 0, 10), ("w", 0, 11)], 0, final=False)
    t.tx(DEV, D | 1, [("r", 0, 11), ("w", 0, 12)], 1, final=False)
    t.tx(HOST, 1, [("r", 0, 10), ("w", 0, 20)], 1)  # FavorHost: host wins
    init = np.array([10], np.uint64)
    assert O.check_p1(t.events(), init).verdict == O.CHECK_PASS
    assert O.check_p2dagger(t.events(), init).verdict == O.CHECK_PASS


def test_unexplained_speculation_fails_p2dagger():
    t = TB()
    t.begin_round(0)
    t.tx(DEV, D | 0, [("r", 0, 77)], 0, final=False)  # 77 was never written by anyone
    t.tx(HOST, 1, [("r", 1, 0), ("w", 1, 5)], 1)
    init = np.array([10, 0], np.uint64)
    assert O.check_p1(t.events(), init).verdict == O.CHECK_PASS  # P1 ignores the aborted side
    r = O.check_p2dagger(t.events(), init)
    assert r.verdict == O.CHECK_FAIL and r.reason == O.REASON_READ and r.got == 77


def test_exhaustive_order_search_for_small_spec_sets():
    """Claimed (ticket) order fails, another order of <= 6 speculative txs explains every read."""
    t = TB()
    t.begin_round(0)
    t.tx(DEV, D | 0, [("r", 0, 2), ("w", 0, 3)], 0, final=False)  # needs D|1 first
    t.tx(DEV, D | 1, [("r", 0, 1), ("w", 0, 2)], 1, final=False)
    init = np.array([1], np.uint64)
    assert O.check_p2dagger(t.events(), init).verdict == O.CHECK_PASS


def test_speculation_after_other_sides_commits_passes():
    """A later device batch that saw a host write applied mid-round: explained with the host's committed txs first."""
    t = TB()
    t.begin_round(0)
    t.tx(HOST, 1, [("r", 0, 1), ("w", 0, 5)], 1)
    t.tx(DEV, D | 0, [("r", 0, 5), ("w", 0, 6)], 0, final=False)
    init = np.array([1], np.uint64)
    assert O.check_p2dagger(t.events(), init).verdict == O.CHECK_PASS


def test_realtime_violation_fails():
    """T2 began after T1's commit but claims an earlier ts."""
    t = TB()
    t.begin_round(0)
    t.tx(HOST, 1, [("r", 0, 0), ("w", 0, 1)], 5)
    t.tx(HOST, 2, [("r", 1, 0), ("w", 1, 1)], 3)
    r = O.check_p1(t.events(), np.zeros(2, np.uint64))
    assert r.verdict == O.CHECK_FAIL and r.reason == O.REASON_REALTIME and r.tx == 2


def test_incomplete_trace():
    t = TB()
    t.begin_round(0)
    t.tx(HOST, 1, [("r", 0, 0), ("w", 0, 1)], 1, final=None)  # speculative commit, no verdict
    r = O.check_p1(t.events(), np.zeros(1, np.uint64))
    assert r.verdict == O.CHECK_INCOMPLETE and r.reason == O.REASON_INCOMPLETE


def test_conflict_aborted_attempts_are_ignored():
    t = TB()
    t.begin_round(0)
    t.add(HOST, O.EV_BEGIN, 7)
    t.add(HOST, O.EV_READ, 7, 0, 12345)  # inconsistent, but the attempt aborted
    t.add(HOST, O.EV_ABORT, 7, 0, O.ABORT_CONFLICT)
    t.tx(HOST, 8, [("r", 0, 0), ("w", 0, 1)], 1)
    assert O.check_p1(t.events(), np.zeros(1, np.uint64)).verdict == O.CHECK_PASS


def test_trace_dump_load_round_trip(tmp_path):
    """trace.hpp: concurrent append with one global seq; dump -> load bit-exact;
    the Python reader parses the same file."""
    exe = os.path.join(ROOT, "build", "trace_format_test")
    if not os.path.exists(exe):
        pytest.skip("build/trace_format_test not built (run __graft_entry__.build())")
    path = str(tmp_path / "t.hetmtrace")
    out = subprocess.run([exe, path], capture_output=True, text=True, timeout=120)
    assert out.returncode == 0, out.stdout + out.stderr
    header, ev = O.load_trace(path)
    assert header["version"] == 1 and header["sizeWords"] == 4096 and header["config"]["threads"] == 8
    assert (np.diff(ev["seq"].astype(np.int64)) == 1).all() and ev["seq"][0] == 0
    assert len(ev) == int(out.stdout.split()[-1])
    # per thread the events keep program order (value = per-thread counter)
    for th in range(8):
        v = ev["value"][((ev["tx"] >> 40) == th) & (ev["kind"] != O.EV_ROUND)]
        assert (np.diff(v.astype(np.int64)) == 1).all()
