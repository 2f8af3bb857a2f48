"""Python mirror of the reference HeTM API for the GPU-side path.

Names follow the reference (SPEC.md op names in the docstrings; error classes
per proj/include/hetm/types.hpp:35-49).  Every call goes through the C-ABI in
libhetm_b200.so; there is no CPU fallback.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from ._lib import lib

# ------------------------------------------------------------------ constants
REPLICA_HOST, REPLICA_DEV, REPLICA_DEV_SHADOW, REPLICA_HOST_SNAPSHOT = 0, 1, 2, 3  # types.hpp:21
BMP_RS, BMP_WS, BMP_CHUNK = 0, 1, 2
APPLY, VALIDATE_ONLY = 0, 1
RETAIN = 0x100  # validate_dptr mode flag: entries join the round arena (capi.h HETM_RETAIN)
KERNEL_BANK, KERNEL_RW, KERNEL_CACHE = 1, 2, 3
TRACE_TX_WORDS = 12  # capi.h HETM_TRACE_TX_WORDS
SCHED_OPTIMISTIC, SCHED_SCAN, SCHED_AUTO = 0, 1, 2  # capi.h HETM_SCHED_* (bank batch schedule)
FAULT_SKIP_RS, FAULT_SKIP_TS, FAULT_SKIP_ROLLBACK = 1, 2, 4  # capi.h HETM_FAULT_* (checker mutation suite)
CACHE_GET, CACHE_SET = 0, 1
CACHE_MISS, CACHE_HIT, CACHE_UPDATED, CACHE_INSERTED, CACHE_EVICTED = range(5)
CACHE_WAYS, CACHE_WAY_WORDS, CACHE_SET_WORDS = 8, 8, 64
CLEAR_RESET_TS = 1
CLEAR_ASYNC = 2
CFG_NO_SHADOW = 1
CFG_L2_FETCH_32 = 2
CFG_MERGE_DELTA = 4
CFG_DETERMINISTIC = 8
H2D, D2H, D2D = 0, 1, 2  # BusDir, bus.hpp:16
TAG_LOG, TAG_MERGE, TAG_SHADOW, TAG_ROLLBACK, TAG_INPUT, TAG_OUTPUT, TAG_RAW, TAG_MERGE_DELTA = range(8)

# 24-byte <addr,value,ts> (write_log.hpp:16-25)
LOG_ENTRY = np.dtype([("addr", "<u8"), ("value", "<u8"), ("ts", "<u8")])
BANK_TX = np.dtype([("acct", "<u4", (4,)), ("amount", "<u8")])
RW_TX = np.dtype(
    [("nr", "<u4"), ("nw", "<u4"), ("r_addr", "<u8", (4,)), ("w_addr", "<u8", (2,)), ("add", "<u8", (2,))]
)
CACHE_TX = np.dtype([("op", "<u4"), ("reserved", "<u4"), ("key", "<u8", (2,)), ("value", "<u8", (4,))])
CACHE_RESULT = np.dtype([("value", "<u8", (4,)), ("status", "<u4"), ("way", "<u4")])
assert LOG_ENTRY.itemsize == 24 and BANK_TX.itemsize == 24 and RW_TX.itemsize == 72
assert CACHE_TX.itemsize == 56 and CACHE_RESULT.itemsize == 40


# --------------------------------------------------------------------- errors
class HetmError(RuntimeError):
    """hetm::HetmError (types.hpp:35)."""

    code = -1


class InvalidSizeError(HetmError): code = 1
class OutOfBoundsError(HetmError): code = 2
class RoundClosedError(HetmError): code = 3
class KernelNotRegisteredError(HetmError): code = 4
class LivelockError(HetmError): code = 5
class NoImplementationError(HetmError): code = 6
class BadAffinityError(HetmError): code = 7
class IncompleteTraceError(HetmError): code = 8
class NondeterministicInputError(HetmError): code = 9
class ConfigError(HetmError): code = 10
class IoError(HetmError): code = 11
class InvalidArgumentError(HetmError): code = 100
class CudaError(HetmError): code = 101
class NoDeviceError(HetmError): code = 102
class NonMonotoneTsError(HetmError): code = 103
class StateError(HetmError): code = 104


_ERRORS = {c.code: c for c in HetmError.__subclasses__()}


def check(rc: int, dev=None) -> None:
    if rc == 0:
        return
    msg = lib.hetm_strerror(rc).decode()
    if dev is not None and rc == CudaError.code:
        msg += ": " + lib.hetm_dev_last_error(dev).decode()
    raise _ERRORS.get(rc, HetmError)(msg)


def device_count() -> int:
    n = C.c_int(0)
    rc = lib.hetm_device_count(C.byref(n))
    return n.value if rc == 0 else 0


def _ptr(a: np.ndarray) -> int:
    assert a.flags["C_CONTIGUOUS"], "arrays crossing the C-ABI must be contiguous"
    return a.ctypes.data


# -------------------------------------------------------------- host helpers
class PinnedArray:
    """Page-locked host buffer (cudaHostAlloc) viewed as a numpy array."""

    def __init__(self, shape, dtype):
        dtype = np.dtype(dtype)
        n = int(np.prod(shape)) * dtype.itemsize
        p = C.c_void_p()
        check(lib.hetm_host_alloc(max(n, 8), C.byref(p)))
        self._p = p
        buf = (C.c_char * max(n, 8)).from_address(p.value)
        self.array = np.frombuffer(buf, dtype=np.uint8, count=n).view(dtype).reshape(shape)

    def free(self):
        if self._p is not None and self._p.value:
            lib.hetm_host_free(self._p)
        self._p = None

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass


def gen_bank_batch(seed: int, n: int, lo: int, span: int, out: np.ndarray | None = None,
                   zipf: float = 0.0) -> np.ndarray:
    """Seeded bank transfers (4 distinct accounts in [lo, lo+span), amount in [1,100]);
    zipf > 0 draws accounts as lo + Zipf(zipf) rank - 1."""
    out = np.empty(n, BANK_TX) if out is None else out
    check(lib.hetm_gen_bank_batch_zipf(seed, n, lo, span, float(zipf), _ptr(out)))
    return out


def gen_host_log(seed: int, n_tx: int, writes_per_tx: int, n_threads: int, lo: int, span: int,
                 ts_base: int = 0, out: np.ndarray | None = None, zipf: float = 0.0) -> np.ndarray:
    """Seeded host write log in WriteLog::allEntries order (thread-major); zipf > 0
    draws the written words as lo + Zipf(zipf) rank - 1."""
    out = np.empty(n_tx * writes_per_tx, LOG_ENTRY) if out is None else out
    check(lib.hetm_gen_host_log_zipf(seed, n_tx, writes_per_tx, n_threads, lo, span, ts_base, float(zipf),
                                     _ptr(out)))
    return out


def gen_cache_batch(seed: int, n: int, key_space: int, alpha: float = 0.5, get_permille: int = 900,
                    part: int = 1, steal_permille: int = 0, out: np.ndarray | None = None) -> np.ndarray:
    """Seeded MemcachedGPU-style GET/SET transactions (BASELINE configs[3]): key
    rank ~ Zipf(alpha), routed to `part` by the key's last bit (part < 0: part 1,
    stealing part-0 keys with probability steal_permille/1000)."""
    out = np.empty(n, CACHE_TX) if out is None else out
    check(lib.hetm_gen_cache_batch(seed, n, key_space, float(alpha), get_permille, part, steal_permille, _ptr(out)))
    return out


def ipc_get_handle(dptr: int) -> bytes:
    """64-byte CUDA IPC handle of a device allocation (cross-process peer access)."""
    buf = (C.c_char * 64)()
    check(lib.hetm_ipc_get_handle(dptr, buf))
    return bytes(buf)


def ipc_open_handle(handle: bytes) -> int:
    p = C.c_void_p()
    check(lib.hetm_ipc_open_handle(C.create_string_buffer(handle, 64), C.byref(p)))
    return p.value


def ipc_close(dptr: int):
    check(lib.hetm_ipc_close(dptr))


def enable_peer_access(device: int, peer: int):
    check(lib.hetm_enable_peer_access(device, peer))


def cache_set_of(key0: int, key1: int, n_sets: int) -> int:
    return int(lib.hetm_cache_set_of(key0, key1, n_sets))


# ------------------------------------------------------------------ snapshots
@dataclass
class BitmapSnapshot:
    """hetm::BitmapSnapshot (bitmap.hpp:15-23)."""

    granBytes: int
    nBits: int
    words: np.ndarray = field(repr=False)

    def test(self, bit: int) -> bool:
        return bool((int(self.words[bit >> 6]) >> (bit & 63)) & 1)

    def set_bits(self) -> np.ndarray:
        bits = np.unpackbits(self.words.view(np.uint8), bitorder="little")
        return np.flatnonzero(bits[: self.nBits])


@dataclass
class BatchResult:
    tickets: np.ndarray
    n_tx: int
    committed: int
    aborts: int
    livelocked: int
    ticket_first: int
    ticket_end: int
    kernel_ms: float
    results: np.ndarray | None = None  # CACHE_RESULT per transaction (KERNEL_CACHE)
    retried: int = 0  # transactions that committed only after >= 2 aborted attempts


# ------------------------------------------------------------- device guest
class GpuDevice:
    """One B200 holding one STMR shard: the device replica, shadow, TS array,
    RS/WS/ChunkMap bitmaps and the batch-TM locks (Stmr + guest-stm-batch
    + engine device half)."""

    def __init__(self, size_words: int, *, shard_base: int = 0, rs_gran_bytes: int = 1024,
                 chunk_bytes: int = 16384, log_capacity: int = 0,
                 max_attempts: int = 0, device: int = 0, shadow: bool = True, l2_fetch_32: bool = False,
                 merge_delta: bool = False, deterministic: bool = False):
        cfg = _lib.DevConfig()
        lib.hetm_dev_config_default(C.byref(cfg))
        cfg.size_words = size_words
        cfg.shard_base = shard_base
        cfg.rs_gran_bytes = rs_gran_bytes
        cfg.chunk_bytes = chunk_bytes
        cfg.log_capacity = log_capacity
        cfg.max_attempts = max_attempts
        cfg.device = device
        cfg.flags = ((0 if shadow else CFG_NO_SHADOW) | (CFG_L2_FETCH_32 if l2_fetch_32 else 0)
                     | (CFG_MERGE_DELTA if merge_delta else 0) | (CFG_DETERMINISTIC if deterministic else 0))
        h = C.c_void_p()
        check(lib.hetm_dev_open(C.byref(cfg), C.byref(h)))
        self.h = h
        self.size_words = size_words
        self.shard_base = shard_base
        self.rs_gran_bytes = rs_gran_bytes
        self.chunk_bytes = chunk_bytes

    # lifecycle --------------------------------------------------------------
    def close(self):
        if getattr(self, "h", None) is not None and self.h.value:
            lib.hetm_dev_close(self.h)
        self.h = None

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _chk(self, rc):
        check(rc, self.h)

    def info(self) -> _lib.DevInfo:
        o = _lib.DevInfo()
        self._chk(lib.hetm_dev_info_get(self.h, C.byref(o)))
        return o

    # stmr raw ops -------------------------------------------
    def raw_write(self, replica: int, addr: int, value: int):
        self._chk(lib.hetm_dev_raw_write(self.h, replica, addr, value))

    def raw_read(self, replica: int, addr: int) -> int:
        v = C.c_uint64()
        self._chk(lib.hetm_dev_raw_read(self.h, replica, addr, C.byref(v)))
        return v.value

    def upload(self, replica: int, addr: int, words: np.ndarray):
        words = np.ascontiguousarray(words, dtype=np.uint64)
        self._chk(lib.hetm_dev_upload(self.h, replica, addr, _ptr(words), words.size))

    def download(self, replica: int, addr: int = None, n: int = None) -> np.ndarray:
        addr = self.shard_base if addr is None else addr
        n = self.size_words - (addr - self.shard_base) if n is None else n
        out = np.empty(n, np.uint64)
        self._chk(lib.hetm_dev_download(self.h, replica, addr, _ptr(out), n))
        return out

    # guest-stm-batch --------------------------------------
    def register_kernel(self, kernel_id: int):
        self._chk(lib.hetm_dev_register_kernel(self.h, kernel_id))

    def execute_batch(self, kernel_id: int, inputs: np.ndarray, want_tickets: bool = True,
                      results: bool = False) -> BatchResult:
        """executeBatch: returns commit tickets (ascending ticket = serial order);
        results=True also returns the per-transaction CACHE_RESULT records."""
        inputs = np.ascontiguousarray(inputs)
        n = inputs.shape[0]
        tickets = np.empty(n, np.uint64) if want_tickets else None
        res = np.zeros(n, CACHE_RESULT) if results else None
        st = _lib.BatchStats()
        self._chk(lib.hetm_dev_execute_batch_ex(self.h, kernel_id, _ptr(inputs) if n else None,
                                                inputs.dtype.itemsize, n,
                                                _ptr(tickets) if (want_tickets and n) else None,
                                                _ptr(res) if (results and n) else None,
                                                CACHE_RESULT.itemsize if results else 0, C.byref(st)))
        r = BatchResult(tickets, st.n_tx, st.committed, st.aborts, st.livelocked, st.ticket_first,
                        st.ticket_end, st.kernel_ms)
        r.results = res
        r.retried = st.retried
        return r

    def set_cache_geometry(self, base_word: int, n_sets: int):
        """Cache region of KERNEL_CACHE: n_sets (power of two) sets from base_word."""
        self._chk(lib.hetm_dev_set_cache_geometry(self.h, base_word, n_sets))

    def bitmap_stats(self):
        """bitmapStats -> (rsBitsSet, wsBitsSet, chunksDirty)."""
        a, b, c = C.c_uint64(), C.c_uint64(), C.c_uint64()
        self._chk(lib.hetm_dev_bitmap_stats(self.h, C.byref(a), C.byref(b), C.byref(c)))
        return a.value, b.value, c.value

    def snapshot(self, which: int) -> BitmapSnapshot:
        n = C.c_uint64()
        self._chk(lib.hetm_dev_bitmap_words(self.h, which, C.byref(n)))
        out = np.zeros(n.value, np.uint64)
        self._chk(lib.hetm_dev_snapshot_bitmap(self.h, which, _ptr(out), n.value))
        gran = self.chunk_bytes if which == BMP_CHUNK else self.rs_gran_bytes
        nbits = (self.size_words * 8 + gran - 1) // gran
        return BitmapSnapshot(gran, nbits, out)

    def or_bitmap(self, which: int, words: np.ndarray):
        words = np.ascontiguousarray(words, dtype=np.uint64)
        self._chk(lib.hetm_dev_or_bitmap(self.h, which, _ptr(words), words.size))

    # interconnect + validation --------------------
    def open_intake(self):
        self._chk(lib.hetm_dev_open_intake(self.h))

    def close_intake(self):
        self._chk(lib.hetm_dev_close_intake(self.h))

    def stream_chunk(self, entries: np.ndarray, src_thread: int = 0, seq: int = 0, mode: int = APPLY):
        """streamChunk + validateChunk.  The buffer must stay alive until round_verdict."""
        entries = np.ascontiguousarray(entries, dtype=LOG_ENTRY)
        self._chk(lib.hetm_dev_stream_chunk(self.h, _ptr(entries) if entries.size else None, entries.size,
                                            src_thread, seq, mode))
        return entries

    def stream_chunk_ex(self, entries: np.ndarray, src_thread: int = 0, seq: int = 0, mode: int = APPLY):
        """streamChunk returning its Delivery (bus.hpp:51-56): the buffer is the
        caller's again once ``delivery_done(d.handle)``."""
        assert entries.flags.c_contiguous and entries.dtype == LOG_ENTRY, "pass the buffer itself (no copy)"
        d = _lib.Delivery()
        self._chk(lib.hetm_dev_stream_chunk_ex(self.h, _ptr(entries) if entries.size else None, entries.size,
                                               src_thread, seq, mode, C.byref(d)))
        return d

    def delivery_done(self, handle: int) -> bool:
        c = C.c_int()
        self._chk(lib.hetm_dev_delivery_done(self.h, handle, C.byref(c)))
        return bool(c.value)

    def delivery_wait(self, handle: int):
        self._chk(lib.hetm_dev_delivery_wait(self.h, handle))

    def source_stats(self, src_thread: int) -> _lib.SourceStats:
        st = _lib.SourceStats()
        self._chk(lib.hetm_dev_source_stats(self.h, src_thread, C.byref(st)))
        return st

    def set_validation_period(self, k: int):
        """Early validation every k VALIDATE_ONLY chunks (default 8)."""
        self._chk(lib.hetm_dev_set_validation_period(self.h, k))

    def apply_log(self):
        self._chk(lib.hetm_dev_apply_log(self.h))

    def poll_conflict(self) -> bool:
        c = C.c_int()
        self._chk(lib.hetm_dev_poll_conflict(self.h, C.byref(c)))
        return bool(c.value)

    def round_verdict(self) -> bool:
        c = C.c_int()
        self._chk(lib.hetm_dev_round_verdict(self.h, C.byref(c)))
        return bool(c.value)

    def sync(self):
        self._chk(lib.hetm_dev_sync(self.h))

    # merge -----------------------------------------------
    def merge_commit(self, host_replica: np.ndarray) -> _lib.MergeStats:
        st = _lib.MergeStats()
        self._chk(lib.hetm_dev_merge_commit(self.h, _ptr(host_replica), C.byref(st)))
        return st

    def merge_abort_device(self, host_replica: np.ndarray | None, optimized: bool = True) -> _lib.MergeStats:
        st = _lib.MergeStats()
        self._chk(lib.hetm_dev_merge_abort_device(self.h, int(optimized),
                                                  None if host_replica is None else _ptr(host_replica),
                                                  C.byref(st)))
        return st

    def merge_abort_host(self, host_replica: np.ndarray, host_snapshot: np.ndarray) -> _lib.MergeStats:
        st = _lib.MergeStats()
        self._chk(lib.hetm_dev_merge_abort_host(self.h, _ptr(host_replica), _ptr(host_snapshot), C.byref(st)))
        return st

    def merge_wait(self):
        self._chk(lib.hetm_dev_merge_wait(self.h))

    def clear_round(self, reset_ts: bool = False, asynchronous: bool = False):
        flags = (CLEAR_RESET_TS if reset_ts else 0) | (CLEAR_ASYNC if asynchronous else 0)
        self._chk(lib.hetm_dev_clear_round(self.h, flags))

    # transferLog (bus.hpp:84-91) ---------------------------------------------
    def transfer_log(self) -> list[tuple[int, int, int]]:
        n = C.c_uint64()
        self._chk(lib.hetm_dev_transfer_count(self.h, C.byref(n)))
        recs = (_lib.TransferRecord * max(n.value, 1))()
        self._chk(lib.hetm_dev_transfer_log(self.h, recs, n.value, C.byref(n)))
        return [(r.dir, r.tag, r.bytes) for r in recs[: n.value]]

    def clear_transfer_log(self):
        self._chk(lib.hetm_dev_clear_transfer_log(self.h))

    # device-resident entries (benchmark / shard router) ---------------------
    def execute_batch_dptr(self, kernel_id: int, d_inputs: int, n: int, d_tickets: int, stream: int = 0,
                           d_results: int = 0):
        self._chk(lib.hetm_dev_execute_batch_dptr_ex(self.h, kernel_id, d_inputs, n, d_tickets, d_results or None,
                                                     stream or None))

    def validate_dptr(self, d_entries: int, n: int, mode: int = APPLY, stream: int = 0):
        self._chk(lib.hetm_dev_validate_dptr(self.h, d_entries, n, mode, stream or None))

    def route_log_dptr(self, d_in: int, n: int, n_shards: int, shard_words: int, d_out: int, d_counts: int,
                       stream: int = 0):
        self._chk(lib.hetm_dev_route_log_dptr(self.h, d_in, n, n_shards, shard_words, d_out, d_counts,
                                              stream or None))

    # fused route + delivery over peer memory ----------------
    def recv_arena(self, n_shards: int, cap: int):
        """(entries, counts) device pointers of this shard's double receive arena."""
        e, c = C.c_void_p(), C.c_void_p()
        self._chk(lib.hetm_dev_recv_arena(self.h, n_shards, cap, C.byref(e), C.byref(c)))
        return e.value, c.value

    def route_to_peers_dptr(self, d_in: int, n: int, n_shards: int, shard_words: int, my_shard: int, cap: int,
                            parity: int, peer_entries, peer_counts, stream: int = 0):
        pe = (C.c_void_p * n_shards)(*peer_entries)
        pc = (C.c_void_p * n_shards)(*peer_counts)
        self._chk(lib.hetm_dev_route_to_peers_dptr(self.h, d_in, n, n_shards, shard_words, my_shard, cap, parity,
                                                   pe, pc, stream or None))

    def apply_received(self, parity: int, mode: int = APPLY, stream: int = 0, count: bool = True):
        """Validate/apply arena[parity]; count=False keeps it asynchronous (returns None)."""
        if not count:
            self._chk(lib.hetm_dev_apply_received(self.h, parity, mode, None, stream or None))
            return None
        n = C.c_uint64()
        self._chk(lib.hetm_dev_apply_received(self.h, parity, mode, C.byref(n), stream or None))
        return n.value

    def read_counters(self):
        c = C.c_int()
        st = _lib.BatchStats()
        self._chk(lib.hetm_dev_read_counters(self.h, C.byref(c), C.byref(st)))
        return bool(c.value), st

    def stream_handle(self, which: int) -> int:
        s = C.c_void_p()
        self._chk(lib.hetm_dev_stream_handle(self.h, which, C.byref(s)))
        return s.value or 0

    def trace_next_batch(self, out: np.ndarray):
        """Arm a checker trace of the next execute_batch (bank / rw): `out` (uint64,
        n_tx * TRACE_TX_WORDS, kept alive by the caller) receives per transaction
        {ticket, read values, rmw read values, written values, 3 reserved}."""
        assert out.dtype == np.uint64 and out.flags["C_CONTIGUOUS"]
        self._trace_keep = out
        self._chk(lib.hetm_dev_trace_next_batch(self.h, out.ctypes.data))

    def merge_stage(self):
        """Device half of mergeCommit, asynchronous (capi.h hetm_dev_merge_stage)."""
        self._chk(lib.hetm_dev_merge_stage(self.h))

    def merge_prepare(self, host_replica: np.ndarray | None = None):
        """Stage the round's delta merge right after the execution phase; with the host
        replica also apply it speculatively (undone by an abort).  See capi.h."""
        if host_replica is not None:
            assert host_replica.dtype == np.uint64 and host_replica.flags["C_CONTIGUOUS"]
            self._prep_keep = host_replica
        self._chk(lib.hetm_dev_merge_prepare(self.h, host_replica.ctypes.data if host_replica is not None else None))

    def bitmap_dptr(self, which: int):
        """(device pointer, n_words) of bitmap `which` (for CUDA IPC export)."""
        p, n = C.c_void_p(), C.c_uint64()
        self._chk(lib.hetm_dev_bitmap_dptr(self.h, which, C.byref(p), C.byref(n)))
        return p.value, n.value

    def bitmap_or_peers(self, which: int, peer_ptrs, word_lo: int = 0, word_hi: int = 0, stream: int = 0):
        """OR words [word_lo, word_hi) (0: all) of the peers' bitmaps into this one (NVLink peer loads)."""
        arr = (C.c_void_p * max(len(peer_ptrs), 1))(*[C.c_void_p(p) for p in peer_ptrs])
        self._chk(lib.hetm_dev_bitmap_or_peers(self.h, which, arr, len(peer_ptrs), word_lo, word_hi, stream or None))

    def set_schedule(self, mode: int):
        """Bank batch schedule: SCHED_OPTIMISTIC | SCHED_SCAN | SCHED_AUTO (default)."""
        self._chk(lib.hetm_dev_set_schedule(self.h, mode))

    def set_fault(self, flags: int):
        """Checker mutation suite only: FAULT_SKIP_RS | FAULT_SKIP_TS | FAULT_SKIP_ROLLBACK."""
        self._chk(lib.hetm_dev_set_fault(self.h, flags))

    def set_timing(self, on: bool = True):
        self._chk(lib.hetm_dev_set_timing(self.h, int(on)))

    def timing(self, which: int):
        """(total_ms, launches) of batch (0) or validation (1) kernels since the last call."""
        t, c = C.c_double(), C.c_uint64()
        self._chk(lib.hetm_dev_timing(self.h, which, C.byref(t), C.byref(c)))
        return t.value, c.value

    def flush_l2(self, stream: int = 0):
        self._chk(lib.hetm_dev_flush_l2(self.h, stream or None))

    # reference op-name aliases -------------------------------------
    rawWrite = raw_write
    rawRead = raw_read
    executeBatch = execute_batch
    bitmapStats = bitmap_stats
    streamChunk = stream_chunk
    mergeCommit = merge_commit
    mergeAbortDevice = merge_abort_device
    mergeAbortHost = merge_abort_host
    clearRound = clear_round
