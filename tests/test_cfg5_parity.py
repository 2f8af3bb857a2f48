"""BASELINE configs[4] at size: validate + TS-guarded apply of CPU write logs of
more than 1 GiB into one 32 GiB STMR shard (the G = 2 geometry of the 64 GiB
configuration; no shadow), bit-exact against the oracle's validateChunk
(oracle/hetm_oracle.c).

The oracle runs on the ADDRESS-COMPACTED round: validateChunk is independent
per word, so mapping every logged word to its rank among the distinct logged
words (and its RS granule bit to a gran-8 bit of that rank) preserves verdict
and apply results exactly while the oracle's STMR shrinks from 2^32 words to
the ~10^8 touched ones.  Every one of the 2^32 device words is then compared:
logged words against the oracle, all others against their initial zero.

Two rounds on the same shard:
  (a) 48 M entries (1.15 GB of log, 24 M two-write transactions, 8 thread
      logs) in ONE apply launch;
  (b) 16 M entries with 10 % of the transactions redirected onto a 2^16-word
      hot set (~26 writers per hot word: TS freshness under races,
      the restore queue at size), delivered as 8 per-thread chunks in shuffled
      order, one launch each (cross-launch freshness, FIFO per source)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

W = 1 << 32  # 32 GiB of STMR words (64 GiB of 16-B cells)
GRAN = 1024
PIECE = 1 << 28  # words per verification download (2 GiB)


def _rs_bits(rs_words, addr):
    b = (addr * np.uint64(8)) // np.uint64(GRAN)
    return ((rs_words[(b >> np.uint64(6)).astype(np.int64)] >> (b & np.uint64(63))) & np.uint64(1)).astype(bool)


def _compact(log, uniq):
    c = log.copy()
    c["addr"] = np.searchsorted(uniq, log["addr"]).astype(np.uint64)
    return c


def test_cfg5_shard_validate_apply_at_size(hetm, orc):
    torch = pytest.importorskip("torch")
    free, _ = torch.cuda.mem_get_info()
    if free < (W * 16 + (W * 8 >> 3) + (8 << 30)):
        pytest.skip(f"needs ~{(W * 24) >> 30} GiB of device memory, {free >> 30} GiB free")

    # ---- logs (product generator: per-thread ts order, distinct words per tx)
    log_a = hetm.gen_host_log(501, 24 << 20, 2, 8, 0, W, ts_base=0)
    n_tx_b = 8 << 20
    log_b = hetm.gen_host_log(502, n_tx_b, 2, 8, 0, W, ts_base=1 << 40)
    hot_base = 3 << 30
    hot = hetm.gen_host_log(503, n_tx_b // 10, 2, 1, hot_base, 1 << 16)  # distinct hot pairs per tx
    rng = np.random.default_rng(504)
    tx_hot = rng.choice(n_tx_b, n_tx_b // 10, replace=False)  # tx k occupies entries 2k, 2k+1
    log_b["addr"][2 * tx_hot] = hot["addr"][0::2]
    log_b["addr"][2 * tx_hot + 1] = hot["addr"][1::2]
    assert log_a.size * 24 > (1 << 30)

    # RS bitmap at density 1e-3 of its bits
    nbits = W * 8 // GRAN
    bits = rng.integers(0, nbits, nbits // 1000).astype(np.uint64)
    rs = np.zeros((nbits + 63) // 64, np.uint64)
    np.bitwise_or.at(rs, (bits >> np.uint64(6)).astype(np.int64), np.left_shift(np.uint64(1), bits & np.uint64(63)))

    # ---- device: round (a) in one launch, round (b) as 8 shuffled per-thread chunks
    per_b = log_b.size // 8
    order_b = rng.permutation(8)
    with hetm.GpuDevice(W, rs_gran_bytes=GRAN, shadow=False, log_capacity=1 << 20) as d:
        d.or_bitmap(hetm.BMP_RS, rs)
        t_a = torch.from_numpy(log_a.view(np.int64).reshape(-1, 3)).cuda()
        d.validate_dptr(t_a.data_ptr(), log_a.size, hetm.APPLY)
        conflict_a = d.round_verdict()
        del t_a
        d.clear_round()  # TS kept (monotone clock), floor rolled; RS cleared
        d.or_bitmap(hetm.BMP_RS, rs)
        t_b = torch.from_numpy(log_b.view(np.int64).reshape(-1, 3)).cuda()
        for t in order_b:
            d.validate_dptr(t_b[t * per_b:(t + 1) * per_b].data_ptr(), per_b, hetm.APPLY)
        conflict_b = d.round_verdict()
        del t_b
        torch.cuda.empty_cache()

        # ---- oracle on the compacted rounds
        uniq = np.unique(np.concatenate([log_a["addr"], log_b["addr"]]))
        U = uniq.size
        rs_c_bits = _rs_bits(rs, uniq)
        rs_c = np.zeros((U + 63) // 64, np.uint64)
        np.bitwise_or.at(rs_c, (np.nonzero(rs_c_bits)[0] >> 6),
                         np.left_shift(np.uint64(1), (np.nonzero(rs_c_bits)[0] & 63).astype(np.uint64)))
        ts_c = np.zeros(U, np.uint64)
        ref_c = np.zeros(U, np.uint64)
        want_a = orc.validate_chunk(_compact(log_a, uniq), rs_c, 8, ts_c, ref_c)
        cb = _compact(log_b, uniq)
        want_b = False
        for t in order_b:
            want_b |= orc.validate_chunk(cb[t * per_b:(t + 1) * per_b], rs_c, 8, ts_c, ref_c)
        assert conflict_a == want_a and conflict_b == want_b
        assert want_a == bool(_rs_bits(rs, log_a["addr"]).any())  # independent brute-force verdict

        # ---- every device word: logged ones == oracle, the rest still zero
        for lo in range(0, W, PIECE):
            got = d.download(hetm.REPLICA_DEV, lo, PIECE)
            i0, i1 = np.searchsorted(uniq, [lo, lo + PIECE])
            want = np.zeros(PIECE, np.uint64)
            want[(uniq[i0:i1] - np.uint64(lo)).astype(np.int64)] = ref_c[i0:i1]
            bad = np.nonzero(got != want)[0]
            assert bad.size == 0, f"{bad.size} words differ in [{lo}, {lo + PIECE}), first at {lo + int(bad[0])}"
        # the hot set is fully covered by the logged words (every hot word was checked above)
        hot_idx = np.searchsorted(uniq, np.arange(hot_base, hot_base + (1 << 16), dtype=np.uint64))
        assert (uniq[hot_idx] == np.arange(hot_base, hot_base + (1 << 16), dtype=np.uint64)).all()
