"""oracle — CPU checker for the Speculative HeTM GPU-side path.

TEST INFRASTRUCTURE ONLY: only tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / `--impl reference` arm may import this package.  The product
(paper_1905_00661_b200) never imports it.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "liboracle.so")
REF_LIB_PATH = os.path.join(HERE, "_ref", "libhetm_ref.so")

ENTRY = np.dtype([("addr", "<u8"), ("value", "<u8"), ("ts", "<u8")])
BANK_TX = np.dtype([("acct", "<u4", (4,)), ("amount", "<u8")])
RW_TX = np.dtype([("nr", "<u4"), ("nw", "<u4"), ("r_addr", "<u8", (4,)), ("w_addr", "<u8", (2,)),
                  ("add", "<u8", (2,))])
CACHE_TX = np.dtype([("op", "<u4"), ("reserved", "<u4"), ("key", "<u8", (2,)), ("value", "<u8", (4,))])
CACHE_RESULT = np.dtype([("value", "<u8", (4,)), ("status", "<u4"), ("way", "<u4")])
RANGE = np.dtype([("offset_bytes", "<u8"), ("bytes", "<u8")])


def build():
    import subprocess
    subprocess.check_call(["make", "-s", "-C", HERE, "all"])


if not os.path.exists(LIB_PATH):
    build()

lib = C.CDLL(LIB_PATH)
_v, _u = C.c_void_p, C.c_uint64
for name, res, args in [
    ("orc_splitmix64", _u, [_u]),
    ("orc_rng_fill_next", None, [_u, _u, _v]),
    ("orc_rng_fill_below", None, [_u, _u, _u, _v]),
    ("orc_rng_fill_uniform", None, [_u, _u, _v]),
    ("orc_bits_for_region", _u, [_u, _u]),
    ("orc_valid_gran", C.c_int, [_u]),
    ("orc_bit_of_word", _u, [_u, _u]),
    ("orc_popcount", _u, [_v, _u]),
    ("orc_validate_chunk", C.c_int, [_v, _u, _v, _u, _u, _v, _v, C.c_int]),
    ("orc_brute_force_intersect", C.c_int, [_v, _u, _v, _u, _u, _u]),
    ("orc_bank_replay", None, [_v, _u, _v, _v, _u, _v, _v, _v, _u, _u]),
    ("orc_rw_replay", None, [_v, _u, _v, _v, _u, _v, _v, _v, _u, _u]),
    ("orc_order_by_ticket", _u, [_v, _u, _v]),
    ("orc_coalesce_chunks", _u, [_v, _u, _u, _u, _v, _u]),
    ("orc_apply_log_ts_order", None, [_v, _u, _v, _u]),
    ("orc_gen_bank_batch", None, [_u, _u, _u, _u, _v]),
    ("orc_gen_host_log", None, [_u, _u, C.c_uint32, C.c_uint32, _u, _u, _u, _v]),
    ("orc_gen_bank_batch_zipf", None, [_u, _u, _u, _u, C.c_double, _v]),
    ("orc_gen_host_log_zipf", None, [_u, _u, C.c_uint32, C.c_uint32, _u, _u, _u, C.c_double, _v]),
    ("orc_zipf_fill", None, [_u, _u, _u, C.c_double, _v]),
    ("orc_cache_hash", _u, [_u, _u]),
    ("orc_cache_set_of", _u, [_u, _u, _u]),
    ("orc_cache_replay", None, [_v, _u, _u, _u, _v, _v, _u, _v, _v, _v, _v, _v, _u, _u]),
    ("orc_cache_host_run", _u, [_v, _u, _u, _u, _v, _u, _u, _v, _v]),
    ("orc_gen_cache_batch", None, [_u, _u, _u, C.c_double, C.c_uint32, C.c_int32, C.c_uint32, _v]),
    ("orc_mt_bank_batch", _u, [_v, _u, _u, _v, _u, C.c_int, _u, _v, _v, _v, _v, _u, _u]),
    ("orc_mt_validate_apply", C.c_int, [_v, _u, _v, _u, _u, _v, _v, C.c_int, C.c_int]),
    ("orc_check_p1", C.c_int, [_v, _u, _v, _u, _v]),
    ("orc_check_p2dagger", C.c_int, [_v, _u, _v, _u, _v]),
]:
    f = getattr(lib, name)
    f.restype, f.argtypes = res, args


def P(a):
    """Pointer of a contiguous numpy array (or None)."""
    if a is None:
        return None
    assert a.flags["C_CONTIGUOUS"]
    return a.ctypes.data


def words_for_bits(nbits: int) -> int:
    return (nbits + 63) // 64


# --------------------------------------------------------------- high level
def rng_next(seed, n):
    o = np.empty(n, np.uint64); lib.orc_rng_fill_next(seed, n, P(o)); return o


def rng_below(seed, bound, n):
    o = np.empty(n, np.uint64); lib.orc_rng_fill_below(seed, bound, n, P(o)); return o


def rng_uniform(seed, n):
    o = np.empty(n, np.float64); lib.orc_rng_fill_uniform(seed, n, P(o)); return o


def gen_bank_batch(seed, n, lo, span, zipf=0.0):
    o = np.empty(n, BANK_TX); lib.orc_gen_bank_batch_zipf(seed, n, lo, span, zipf, P(o)); return o


def gen_host_log(seed, n_tx, wpt, threads, lo, span, ts_base=0, zipf=0.0):
    o = np.empty(n_tx * wpt, ENTRY)
    lib.orc_gen_host_log_zipf(seed, n_tx, wpt, threads, lo, span, ts_base, zipf, P(o))
    return o


def gen_cache_batch(seed, n, key_space, alpha=0.5, get_permille=900, part=1, steal_permille=0):
    o = np.empty(n, CACHE_TX)
    lib.orc_gen_cache_batch(seed, n, key_space, alpha, get_permille, part, steal_permille, P(o))
    return o


def cache_replay(stmr, txs, tickets, n_sets, gran, chunk, base=0, cache_base=0):
    """Device batch in ticket order on `stmr` (in place); returns (results, rs, ws, chunk) words."""
    txs = np.ascontiguousarray(txs, CACHE_TX)
    tickets = np.ascontiguousarray(tickets, np.uint64)
    order = order_by_ticket(tickets)
    res = np.zeros(txs.size, CACHE_RESULT)
    W = stmr.size
    rs = np.zeros(words_for_bits(W * 8 // gran), np.uint64)
    ws = np.zeros_like(rs)
    ch = np.zeros(words_for_bits((W * 8 + chunk - 1) // chunk), np.uint64)
    lib.orc_cache_replay(P(stmr), base, cache_base, n_sets, P(txs), P(order), order.size, P(tickets), P(res),
                         P(rs), P(ws), P(ch), gran, chunk)
    return res, rs, ws, ch


def cache_host_run(stmr, txs, n_sets, ts_base, base=0, cache_base=0):
    """Host transactions in order (ts = ts_base+1+i) on `stmr`; returns (results, write log)."""
    txs = np.ascontiguousarray(txs, CACHE_TX)
    res = np.zeros(txs.size, CACHE_RESULT)
    log = np.zeros(txs.size * 8, ENTRY)
    m = lib.orc_cache_host_run(P(stmr), base, cache_base, n_sets, P(txs), txs.size, ts_base, P(res), P(log))
    return res, log[:m].copy()


def zipf_ranks(seed, n, span, alpha):
    o = np.empty(n, np.uint64); lib.orc_zipf_fill(seed, n, span, alpha, P(o)); return o


def validate_chunk(entries, rs_words, gran, ts, dev, apply=True, base=0):
    entries = np.ascontiguousarray(entries, ENTRY)
    return bool(lib.orc_validate_chunk(P(entries), entries.size, P(rs_words), gran, base, P(ts), P(dev), int(apply)))


def brute_force_intersect(entries, rs_words, rs_bits, gran, base=0):
    entries = np.ascontiguousarray(entries, ENTRY)
    return bool(lib.orc_brute_force_intersect(P(entries), entries.size, P(rs_words), rs_bits, gran, base))


def order_by_ticket(tickets):
    tickets = np.ascontiguousarray(tickets, np.uint64)
    o = np.empty(tickets.size, np.uint64)
    m = lib.orc_order_by_ticket(P(tickets), tickets.size, P(o))
    return o[:m]


def bank_replay(stmr, txs, order, gran, chunk, base=0):
    """sequentialReplay of device txs; returns (rs, ws, chunk) bitmaps as word arrays."""
    W = stmr.size
    rs = np.zeros(words_for_bits((W * 8 + gran - 1) // gran), np.uint64)
    ws = np.zeros_like(rs)
    ch = np.zeros(words_for_bits((W * 8 + chunk - 1) // chunk), np.uint64)
    order = np.ascontiguousarray(order, np.uint64)
    lib.orc_bank_replay(P(stmr), base, P(txs), P(order), order.size, P(rs), P(ws), P(ch), gran, chunk)
    return rs, ws, ch


def rw_replay(stmr, txs, order, gran, chunk, base=0):
    W = stmr.size
    rs = np.zeros(words_for_bits((W * 8 + gran - 1) // gran), np.uint64)
    ws = np.zeros_like(rs)
    ch = np.zeros(words_for_bits((W * 8 + chunk - 1) // chunk), np.uint64)
    order = np.ascontiguousarray(order, np.uint64)
    lib.orc_rw_replay(P(stmr), base, P(txs), P(order), order.size, P(rs), P(ws), P(ch), gran, chunk)
    return rs, ws, ch


def coalesce_chunks(chunk_words, n_chunks, chunk_bytes, region_bytes):
    out = np.empty(max(n_chunks, 1), RANGE)
    m = lib.orc_coalesce_chunks(P(chunk_words), n_chunks, chunk_bytes, region_bytes, P(out), out.size)
    return [(int(r["offset_bytes"]), int(r["bytes"])) for r in out[:m]]


def apply_log_ts_order(region, entries, base=0):
    entries = np.ascontiguousarray(entries, ENTRY)
    lib.orc_apply_log_ts_order(P(region), base, P(entries), entries.size)


def mt_bank_batch(stmr, txs, threads, lock_entries=1 << 22, gran=1024, chunk=16384, base=0, tickets=True):
    W = stmr.size
    tk = np.empty(txs.size, np.uint64) if tickets else None
    rs = np.zeros(words_for_bits((W * 8 + gran - 1) // gran), np.uint64)
    ws = np.zeros_like(rs)
    ch = np.zeros(words_for_bits((W * 8 + chunk - 1) // chunk), np.uint64)
    c = lib.orc_mt_bank_batch(P(stmr), base, W, P(txs), txs.size, threads, lock_entries, P(tk), P(rs), P(ws),
                              P(ch), gran, chunk)
    return c, tk, rs, ws, ch


def mt_validate_apply(entries, rs_words, gran, ts, dev, threads, apply=True, base=0):
    entries = np.ascontiguousarray(entries, ENTRY)
    return bool(lib.orc_mt_validate_apply(P(entries), entries.size, P(rs_words), gran, base, P(ts), P(dev),
                                          threads, int(apply)))


# ---- checker (checker.c) ------------------------------------
TRACE_EVENT = np.dtype([("seq", "<u8"), ("tx", "<u8"), ("addr", "<u8"), ("value", "<u8"), ("round", "<u4"),
                        ("device", "u1"), ("kind", "u1"), ("pad", "<u2")])
assert TRACE_EVENT.itemsize == 40
EV_BEGIN, EV_READ, EV_WRITE, EV_SPEC_COMMIT, EV_FINAL_COMMIT, EV_ABORT, EV_ROUND = range(7)
ABORT_CONFLICT, ABORT_ROUND = 1, 2
CHECK_PASS, CHECK_FAIL, CHECK_INCOMPLETE = 0, 1, 2
REASON_NONE, REASON_READ, REASON_REALTIME, REASON_INCOMPLETE, REASON_BAD_ADDR = range(5)


class CheckResult(C.Structure):
    _fields_ = [("verdict", C.c_int), ("reason", C.c_int), ("tx", _u), ("addr", _u), ("expected", _u), ("got", _u),
                ("round", C.c_uint32), ("checked_txs", _u), ("checked_reads", _u)]


def _check(fn, events, init):
    ev = np.ascontiguousarray(events, dtype=TRACE_EVENT)
    st = np.ascontiguousarray(init, dtype=np.uint64)
    r = CheckResult()
    fn(P(ev) if len(ev) else None, len(ev), P(st), len(st), C.byref(r))
    return r


def check_p1(events, init):
    """checkP1: the finally committed transactions explained by the claimed serial order."""
    return _check(lib.orc_check_p1, events, init)


def check_p2dagger(events, init):
    """checkP2dagger: speculative commits of aborted sides explained by their own device's order."""
    return _check(lib.orc_check_p2dagger, events, init)


def load_trace(path):
    """Parses a HETMTRC1 dump (include/hetm_b200/trace.hpp): (header dict, events)."""
    import json
    import struct
    raw = open(path, "rb").read()
    if raw[:8] != b"HETMTRC1":
        raise ValueError("not a HETMTRC1 trace")
    (hl,) = struct.unpack_from("<I", raw, 8)
    header = json.loads(raw[12:12 + hl].decode())
    body = raw[12 + hl:]
    rec = 4 + TRACE_EVENT.itemsize
    if len(body) % rec:
        raise ValueError("truncated trace record")
    recs = np.frombuffer(body, dtype=np.uint8).reshape(-1, rec)
    if len(recs) and not (recs[:, :4].copy().view("<u4") == TRACE_EVENT.itemsize).all():
        raise ValueError("bad record length")
    return header, recs[:, 4:].copy().view(TRACE_EVENT).reshape(-1)


def load_ref():
    """The reference-header shim (oracle/_ref), present only where /root/reference was."""
    if not os.path.exists(REF_LIB_PATH):
        return None
    r = C.CDLL(REF_LIB_PATH)
    for name, res, args in [
        ("ref_rng_next", None, [_u, _u, _v]),
        ("ref_rng_below", None, [_u, _u, _u, _v]),
        ("ref_rng_uniform", None, [_u, _u, _v]),
        ("ref_splitmix64", _u, [_u]),
        ("ref_access_bitmap", C.c_longlong, [_u, _u, _v, _u, _v]),
        ("ref_chunk_map", C.c_longlong, [_u, _u, _v, _u, _v, _u]),
        ("ref_write_log_all", None, [_v, _v, _u, C.c_int, _v]),
        ("ref_log_entry_bytes", _u, []),
    ]:
        f = getattr(r, name)
        f.restype, f.argtypes = res, args
    return r
