"""The oracle, pinned: against the reference headers' golden vectors and the
SPEC.md examples / acceptance properties on the hot path.  CPU only."""
import itertools
import json
import os

import numpy as np
import pytest

import oracle as O

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "ref_vectors.json")))


# ------------------------------------------------ golden: reference headers
@pytest.mark.parametrize("rec", GOLD["rng"], ids=lambda r: f"seed{r['seed']}")
def test_detrng_matches_reference(rec):
    """det_rng.hpp:19-42 — next/below/uniform sequences bit-identical."""
    s = rec["seed"]
    assert [int(x) for x in O.rng_next(s, 16)] == rec["next"]
    for bound, want in rec["below"].items():
        assert [int(x) for x in O.rng_below(s, int(bound), 16)] == want
    assert O.rng_uniform(s, 8).tolist() == rec["uniform"]


def test_splitmix64_matches_reference():
    for x, y in GOLD["splitmix64"]:
        assert O.lib.orc_splitmix64(x) == y


def test_appendix_a_kats():
    """SURVEY.md Appendix A (computed from the reference headers)."""
    assert O.rng_next(0, 4).tolist() == [12561902727665508292, 495403393847554056, 18228640026652296647,
                                         2072868329570037522]
    assert O.rng_below(1, 1 << 20, 8).tolist() == [594082, 386074, 727200, 927769, 215235, 1032697, 28552, 900520]


@pytest.mark.parametrize("rec", GOLD["access_bitmap"], ids=lambda r: r["name"])
def test_access_bitmap_geometry_matches_reference(rec):
    """bitmap.hpp:94-124: ceil bit count, bit = addr*8/gran, invalid gran."""
    region, gran = rec["region_bytes"], rec["gran"]
    if rec["nbits"] < 0:
        assert not O.lib.orc_valid_gran(gran)
        return
    assert O.lib.orc_valid_gran(gran)
    nbits = O.lib.orc_bits_for_region(region, gran)
    assert nbits == rec["nbits"]
    words = np.zeros(O.words_for_bits(nbits), np.uint64)
    for a in rec["addrs"]:
        b = O.lib.orc_bit_of_word(a, gran)
        words[b >> 6] |= np.uint64(1 << (b & 63))
    assert words.tolist() == rec["words"]


@pytest.mark.parametrize("rec", GOLD["chunk_map"], ids=lambda r: r["name"])
def test_chunk_map_matches_reference(rec):
    """bitmap.hpp:128-158: dirty chunk set + forEachDirty ascending order."""
    if rec["dirty"] is None:
        assert not O.lib.orc_valid_gran(rec["chunk"])
        return
    dirty = sorted({O.lib.orc_bit_of_word(a, rec["chunk"]) for a in rec["addrs"]})
    assert dirty == rec["dirty"]


def test_write_log_all_entries_thread_order():
    """write_log.hpp:74-82: allEntries concatenates per-thread logs in thread order."""
    wl = GOLD["write_log"]
    per = [[] for _ in range(wl["threads"])]
    for t, e in zip(wl["tid"], wl["entries"]):
        per[t].append(e)
    assert list(itertools.chain(*per)) == wl["all_entries"]
    assert GOLD["log_entry_bytes"] == 24 == O.ENTRY.itemsize


def test_host_log_generator_layout():
    """gen_host_log deals tx i to thread i%T, ts-ordered per thread, shared ts per tx."""
    log = O.gen_host_log(5, 10, 2, 3, 100, 1000, ts_base=40)
    assert log.size == 20
    per_thread = [4, 3, 3]  # txs 0,3,6,9 | 1,4,7 | 2,5,8
    pos = 0
    for t, cnt in enumerate(per_thread):
        chunk = log[pos:pos + 2 * cnt]
        ts = chunk["ts"].reshape(cnt, 2)
        assert (ts[:, 0] == ts[:, 1]).all()
        assert ts[:, 0].tolist() == [41 + t + 3 * k for k in range(cnt)]
        assert (chunk["addr"].reshape(cnt, 2)[:, 0] != chunk["addr"].reshape(cnt, 2)[:, 1]).all()
        pos += 2 * cnt
    assert ((log["addr"] >= 100) & (log["addr"] < 1100)).all()


def test_bank_generator_distinct_accounts():
    txs = O.gen_bank_batch(1, 5000, 0, 64)
    for t in txs:
        assert len(set(t["acct"].tolist())) == 4
    assert (txs["amount"] >= 1).all() and (txs["amount"] <= 100).all()


def test_zipf_sampler_law():
    """10^6 samples at alpha 0.5 -- top-10 rank frequencies within
    5% of the analytic law k^-a / H(N, a) (N = 1000 keeps the top ranks' counts
    large enough that 5% is well above sampling noise)."""
    N, n, a = 1000, 10**6, 0.5
    ranks = O.zipf_ranks(3, n, N, a)
    assert ranks.min() >= 1 and ranks.max() <= N
    H = float(np.sum(np.arange(1, N + 1, dtype=np.float64) ** -a))
    counts = np.bincount(ranks[ranks <= 10].astype(np.int64), minlength=11)[1:]
    expect = n * np.arange(1, 11, dtype=np.float64) ** -a / H
    assert (np.abs(counts - expect) / expect < 0.05).all(), (counts, expect)


@pytest.mark.parametrize("alpha", [0.99, 1.2])
def test_zipf_sampler_law_skewed(alpha):
    N, n = 1 << 20, 10**6
    ranks = O.zipf_ranks(9, n, N, alpha)
    H = float(np.sum(np.arange(1, N + 1, dtype=np.float64) ** -alpha))
    counts = np.bincount(ranks[ranks <= 10].astype(np.int64), minlength=11)[1:]
    expect = n * np.arange(1, 11, dtype=np.float64) ** -alpha / H
    assert (np.abs(counts - expect) / expect < 0.05).all(), (counts, expect)


def test_zipf_bank_batch_distinct_and_hot():
    txs = O.gen_bank_batch(5, 20000, 100, 1 << 20, zipf=0.99)
    acct = txs["acct"].astype(np.int64)
    assert (np.sort(acct, axis=1)[:, 1:] != np.sort(acct, axis=1)[:, :-1]).all()  # distinct per tx
    assert acct.min() >= 100 and acct.max() < 100 + (1 << 20)
    assert (acct == 100).any(axis=1).mean() > 0.1  # rank 1 is hot


def test_cache_lru_matches_independent_model():
    """within one set the evicted way is always the least recently
    touched -- the oracle's stamp-based LRU vs a recency-list model."""
    n_sets, n = 4, 3000
    txs = O.gen_cache_batch(5, n, 200, alpha=0.3, get_permille=600, part=1)
    stmr = np.zeros(n_sets * 64, np.uint64)
    res, log = O.cache_host_run(stmr, txs, n_sets, ts_base=0)
    sets = {}  # set -> list of (key, value) with most recent last, <= 8 entries
    for i, t in enumerate(txs):
        key = (int(t["key"][0]), int(t["key"][1]))
        s = int(O.lib.orc_cache_set_of(key[0], key[1], n_sets))
        lst = sets.setdefault(s, [])
        idx = next((j for j, (k, _) in enumerate(lst) if k == key), None)
        if t["op"] == 0:
            if idx is None:
                assert res[i]["status"] == 0
            else:
                assert res[i]["status"] == 1 and tuple(res[i]["value"]) == lst[idx][1]
                lst.append(lst.pop(idx))
        else:
            val = tuple(int(x) for x in t["value"])
            if idx is not None:
                assert res[i]["status"] == 2
                lst.pop(idx)
            elif len(lst) < 8:
                assert res[i]["status"] == 3
            else:
                assert res[i]["status"] == 4
                lst.pop(0)  # least recently touched
            lst.append((key, val))
    assert (res["status"] == 4).sum() > 100  # evictions exercised
    # the host write log replays to the same region
    again = np.zeros_like(stmr)
    O.apply_log_ts_order(again, log)
    assert (again == stmr).all()


# --------------------------------------------------- SPEC.md examples (KATs)
def _rs(nbits, bits):
    w = np.zeros(O.words_for_bits(nbits), np.uint64)
    for b in bits:
        w[b >> 6] |= np.uint64(1 << (b & 63))
    return w


def _entries(rows):
    return np.array(rows, dtype=O.ENTRY)


def test_validate_spec_351_apply_fresh():
    """SPEC.md:351 RS clear, TS 0, ts 5 -> applied, TS=5, no conflict."""
    W, gran = 64, 8
    rs, ts, dev = _rs(64, []), np.zeros(W, np.uint64), np.zeros(W, np.uint64)
    assert not O.validate_chunk(_entries([(3, 99, 5)]), rs, gran, ts, dev)
    assert dev[3] == 99 and ts[3] == 5


@pytest.mark.parametrize("order", [(0, 1), (1, 0)])
def test_validate_spec_352_max_ts_any_order(order):
    """SPEC.md:352 two entries ts 7 then 3, any order -> ts-7 value."""
    rows = [(4, 700, 7), (4, 300, 3)]
    rs, ts, dev = _rs(64, []), np.zeros(64, np.uint64), np.zeros(64, np.uint64)
    for i in order:
        O.validate_chunk(_entries([rows[i]]), rs, 8, ts, dev)
    assert dev[4] == 700 and ts[4] == 7


def test_validate_spec_353_conflict_still_applied():
    """SPEC.md:353 RS bit set -> conflict, value still applied."""
    rs, ts, dev = _rs(64, [2]), np.zeros(64, np.uint64), np.zeros(64, np.uint64)
    assert O.validate_chunk(_entries([(2, 5, 1)]), rs, 8, ts, dev)
    assert dev[2] == 5


def test_validate_only_skips_apply():
    rs, ts, dev = _rs(64, [2]), np.zeros(64, np.uint64), np.zeros(64, np.uint64)
    assert O.validate_chunk(_entries([(2, 5, 1)]), rs, 8, ts, dev, apply=False)
    assert dev[2] == 0 and ts[2] == 0


def test_false_positive_1k_granularity():
    """read and write in the same 1024-B bit, different words -> conflict."""
    W, gran = 1 << 17, 1024
    nbits = W * 8 // gran
    rs = _rs(nbits, [O.lib.orc_bit_of_word(0, gran)])  # device read word 0
    e = _entries([(127, 1, 1)])                           # host wrote word 127 (same 1 KiB)
    ts, dev = np.zeros(W, np.uint64), np.zeros(W, np.uint64)
    assert O.validate_chunk(e, rs, gran, ts, dev, apply=False)
    assert O.brute_force_intersect(e, rs, nbits, gran)
    e2 = _entries([(128, 1, 1)])
    assert not O.brute_force_intersect(e2, rs, nbits, gran)


def test_brute_force_matches_validator_random():
    """1000 random rounds, exact match of the two independent codes."""
    r = np.random.default_rng(3)
    for _ in range(1000):
        W = int(r.integers(64, 4096))
        gran = int(r.choice([8, 64, 1024]))
        nbits = (W * 8 + gran - 1) // gran
        rs = _rs(nbits, r.choice(nbits, size=min(nbits, int(r.integers(0, 4))), replace=False).tolist())
        n = int(r.integers(0, 6))
        e = np.zeros(n, O.ENTRY)
        e["addr"] = r.integers(0, W, n)
        e["ts"] = np.arange(1, n + 1)
        ts, dev = np.zeros(W, np.uint64), np.zeros(W, np.uint64)
        assert O.validate_chunk(e, rs, gran, ts, dev, apply=False) == O.brute_force_intersect(e, rs, nbits, gran)


def test_ts_freshness_permutations():
    """Acceptance #5: duplicate-heavy multi-chunk logs, >=10 permuted
    delivery orders -> every word ends at its max-ts value."""
    r = np.random.default_rng(11)
    W = 32
    log = np.zeros(200, O.ENTRY)
    log["addr"] = r.integers(0, W, 200)
    log["value"] = r.integers(0, 2**63, 200, dtype=np.uint64)
    log["ts"] = r.permutation(200) + 1
    want = np.zeros(W, np.uint64)
    best = np.zeros(W, np.uint64)
    for e in log:
        if e["ts"] > best[e["addr"]]:
            best[e["addr"]], want[e["addr"]] = e["ts"], e["value"]
    chunks = np.array_split(log, 10)
    for _ in range(12):
        ts, dev = np.zeros(W, np.uint64), np.zeros(W, np.uint64)
        for k in r.permutation(len(chunks)):
            O.validate_chunk(chunks[k], _rs(4, []), 8, ts, dev)
        assert (dev == want).all()


def test_coalescing_spec_examples():
    """empty, adjacent, separated, 1 word."""
    C, region = 16384, 1 << 20
    n = region // C
    assert O.coalesce_chunks(_rs(n, []), n, C, region) == []
    assert O.coalesce_chunks(_rs(n, [0, 1]), n, C, region) == [(0, 32768)]
    assert O.coalesce_chunks(_rs(n, [0, 2]), n, C, region) == [(0, C), (2 * C, C)]
    assert O.coalesce_chunks(_rs(n, [5]), n, C, region) == [(5 * C, C)]


def test_rollback_spec_378():
    """device wrote {3,9}; host wrote 3 (read by device) -> after abort
    dev[9] = round start, dev[3] = host value (shadow + ts-ordered host log)."""
    start = np.arange(16, dtype=np.uint64) * 10
    shadow = start.copy()
    O.apply_log_ts_order(shadow, _entries([(3, 777, 4)]))
    assert shadow[9] == start[9] and shadow[3] == 777


def test_ts_order_apply_equals_validate_max():
    r = np.random.default_rng(5)
    W = 50
    log = np.zeros(300, O.ENTRY)
    log["addr"] = r.integers(0, W, 300)
    log["value"] = r.integers(0, 1000, 300)
    log["ts"] = r.permutation(300) + 1
    a = np.zeros(W, np.uint64)
    O.apply_log_ts_order(a, log)
    b, ts = np.zeros(W, np.uint64), np.zeros(W, np.uint64)
    O.validate_chunk(log, _rs(1, []), 8, ts, b)
    assert (a == b).all()


def test_execute_batch_spec_209_bitmaps():
    """1 tx reading word 0, writing word 1 @8 B -> RS{0,1} WS{1}, stats (2,1,1)."""
    tx = np.zeros(1, O.RW_TX)
    tx["nr"], tx["nw"] = 1, 1
    tx["r_addr"][0, 0] = 0
    tx["w_addr"][0, 0] = 1
    stmr = np.zeros(64, np.uint64)
    rs, ws, ch = O.rw_replay(stmr, tx, np.array([0], np.uint64), 8, 16384)
    assert rs[0] == 0x3 and ws[0] == 0x2
    assert (O.lib.orc_popcount(O.P(rs), rs.size), O.lib.orc_popcount(O.P(ws), ws.size),
            O.lib.orc_popcount(O.P(ch), ch.size)) == (2, 1, 1)


def test_bank_replay_sum_invariant_and_ws_subset_rs():
    W = 1 << 12
    txs = O.gen_bank_batch(9, 2000, 0, W)
    stmr = np.full(W, 1000, np.uint64)
    rs, ws, ch = O.bank_replay(stmr, txs, np.arange(2000, dtype=np.uint64), 64, 16384)
    assert int(stmr.sum(dtype=np.uint64)) == 1000 * W
    assert ((ws & ~rs) == 0).all()  # WS subset of RS


@pytest.mark.parametrize("threads", [1, 4])
def test_mt_bank_batch_replays_in_ticket_order(threads):
    """The CPU baseline commits a serializable history: replay in ticket order == its state."""
    W = 1 << 10  # small: heavy contention
    txs = O.gen_bank_batch(4, 20000, 0, W)
    s = np.full(W, 500, np.uint64)
    c, tk, rs, ws, ch = O.mt_bank_batch(s, txs, threads, lock_entries=1 << 8, gran=64)
    assert c == 20000
    order = O.order_by_ticket(tk)
    assert order.size == 20000 and len(np.unique(tk)) == 20000
    ref = np.full(W, 500, np.uint64)
    rs2, ws2, ch2 = O.bank_replay(ref, txs, order, 64, 16384)
    assert (ref == s).all()
    assert (rs == rs2).all() and (ws == ws2).all() and (ch == ch2).all()


def test_mt_validate_apply_matches_serial():
    r = np.random.default_rng(8)
    W, n = 1 << 12, 50000
    log = np.zeros(n, O.ENTRY)
    log["addr"] = r.integers(0, W, n)
    log["value"] = r.integers(0, 2**63, n, dtype=np.uint64)
    log["ts"] = r.permutation(n) + 1
    rs = _rs(W * 8 // 64, [3, 17])
    ts1, d1 = np.zeros(W, np.uint64), np.zeros(W, np.uint64)
    ts2, d2 = np.zeros(W, np.uint64), np.zeros(W, np.uint64)
    c1 = O.validate_chunk(log, rs, 64, ts1, d1)
    c2 = O.mt_validate_apply(log, rs, 64, ts2, d2, 4)
    assert c1 == c2 and (d1 == d2).all() and (ts1 == ts2).all()
