/*
 * hetm_oracle — CPU restatement of the Speculative HeTM GPU-side path.
 *
 * TEST INFRASTRUCTURE ONLY.  This library is the parity checker and the CPU
 * baseline.  Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline
 * leg / `--impl reference` arm may load it.  The product path
 * (paper_1905_00661_b200, libhetm_b200.so) never links or calls it.
 *
 * Every function cites the reference line it restates (paths relative to
 * /root/reference).  The reference mount holds no implementation of the
 * batch TM, validation or merge: those functions restate the
 * behavioural SPEC.md and are pinned by SPEC.md's examples and acceptance
 * properties; the RNG, bitmap geometry and write-log ordering are pinned
 * against the reference headers themselves (oracle/_ref, tests/golden/).
 */
#ifndef HETM_ORACLE_H
#define HETM_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct { uint64_t addr, value, ts; } orc_entry;          /* write_log.hpp:16-22 */
typedef struct { uint32_t acct[4]; uint64_t amount; } orc_bank_tx; /* capi.h hetm_bank_tx */
typedef struct {
    uint32_t nr, nw;
    uint64_t r_addr[4], w_addr[2], add[2];
} orc_rw_tx;                                                       /* capi.h hetm_rw_tx */
typedef struct { uint64_t offset_bytes, bytes; } orc_range;
typedef struct { uint32_t op, reserved; uint64_t key[2]; uint64_t value[4]; } orc_cache_tx; /* capi.h hetm_cache_tx */
typedef struct { uint64_t value[4]; uint32_t status, way; } orc_cache_result;            /* hetm_cache_result */

/* ---- det_rng.hpp:8-42 ---- */
uint64_t orc_splitmix64(uint64_t x);
typedef struct { uint64_t state; } orc_rng;
void orc_rng_init(orc_rng* r, uint64_t seed);
uint64_t orc_rng_next(orc_rng* r);
uint64_t orc_rng_below(orc_rng* r, uint64_t bound);
double orc_rng_uniform(orc_rng* r);
void orc_rng_fill_next(uint64_t seed, uint64_t n, uint64_t* out);
void orc_rng_fill_below(uint64_t seed, uint64_t bound, uint64_t n, uint64_t* out);
void orc_rng_fill_uniform(uint64_t seed, uint64_t n, double* out);

/* ---- bitmap.hpp:94-158 geometry ---- */
uint64_t orc_bits_for_region(uint64_t region_bytes, uint64_t gran_bytes); /* ceil, bitmap.hpp:96-97 */
int orc_valid_gran(uint64_t gran_bytes);                                  /* bitmap.hpp:99-100 */
uint64_t orc_bit_of_word(uint64_t addr, uint64_t gran_bytes);             /* bitmap.hpp:104 */
void orc_bitmap_set(uint64_t* words, uint64_t bit);
int orc_bitmap_test(const uint64_t* words, uint64_t bit);
uint64_t orc_popcount(const uint64_t* words, uint64_t n_words);

/* ---- engine.validateChunk, SPEC.md:345-353 (single worker) ----
 * Addresses are global; `base` is subtracted to index ts/dev/RS (shards).
 * Returns conflictFound.  The caller owns the per-round TS reset. */
int orc_validate_chunk(const orc_entry* e, uint64_t n, const uint64_t* rs_words, uint64_t gran_bytes,
                       uint64_t base, uint64_t* ts, uint64_t* dev, int apply);

/* ---- checker.bruteForceIntersect; shares no code with the
 * validator. ---- */
int orc_brute_force_intersect(const orc_entry* e, uint64_t n, const uint64_t* rs_words,
                              uint64_t rs_bits, uint64_t gran_bytes, uint64_t base);

/* ---- sequentialReplay of device txs + executeBatch
 * bitmap post-condition.  order[k] = index of the k-th tx in
 * serial order (n_order entries; e.g. sorted by commit ticket).  Bitmaps
 * (nullable) are OR-ed. ---- */
void orc_bank_replay(uint64_t* stmr, uint64_t base, const orc_bank_tx* tx, const uint64_t* order,
                     uint64_t n_order, uint64_t* rs, uint64_t* ws, uint64_t* chunks,
                     uint64_t gran_bytes, uint64_t chunk_bytes);
void orc_rw_replay(uint64_t* stmr, uint64_t base, const orc_rw_tx* tx, const uint64_t* order,
                   uint64_t n_order, uint64_t* rs, uint64_t* ws, uint64_t* chunks,
                   uint64_t gran_bytes, uint64_t chunk_bytes);
/* Stable ticket sort: writes tx indices with ticket != UINT64_MAX ordered by
 * ticket into order_out; returns the count. */
uint64_t orc_order_by_ticket(const uint64_t* tickets, uint64_t n, uint64_t* order_out);

/* ---- stmr.copyChunks coalescing, SPEC.md:62-70 / copyDeviceToHost SPEC.md:279-287 ---- */
uint64_t orc_coalesce_chunks(const uint64_t* chunk_words, uint64_t n_chunks, uint64_t chunk_bytes,
                             uint64_t region_bytes, orc_range* out, uint64_t max_out);

/* ---- mergeAbortDevice optimized path: shadow patched by the
 * round's full host log in ts order. ---- */
void orc_apply_log_ts_order(uint64_t* region, uint64_t base, const orc_entry* e, uint64_t n);

/* ---- seeded inputs (generators must match libhetm_b200's) ---- */
void orc_gen_bank_batch(uint64_t seed, uint64_t n, uint64_t lo, uint64_t span, orc_bank_tx* out);
/* alpha > 0: accounts / words drawn as lo + zipf(alpha) rank - 1 (rank 1 hottest) */
void orc_gen_bank_batch_zipf(uint64_t seed, uint64_t n, uint64_t lo, uint64_t span, double alpha, orc_bank_tx* out);
void orc_gen_host_log_zipf(uint64_t seed, uint64_t n_tx, uint32_t wpt, uint32_t T, uint64_t lo, uint64_t span,
                           uint64_t ts_base, double alpha, orc_entry* out);
uint64_t orc_cache_hash(uint64_t k0, uint64_t k1);
uint64_t orc_cache_set_of(uint64_t k0, uint64_t k1, uint64_t n_sets);
/* device batch replayed in ticket order (LRU stamp = ticket + 1) */
void orc_cache_replay(uint64_t* s, uint64_t base, uint64_t cbase, uint64_t n_sets, const orc_cache_tx* tx,
                      const uint64_t* order, uint64_t n_order, const uint64_t* tickets, orc_cache_result* results,
                      uint64_t* rs, uint64_t* ws, uint64_t* ch, uint64_t gran, uint64_t chunk);
/* host transactions in order with ts = ts_base+1+i (LRU stamp = ts); their
 * writes appended to `log` as <addr,value,ts>; returns the entry count */
uint64_t orc_cache_host_run(uint64_t* s, uint64_t base, uint64_t cbase, uint64_t n_sets, const orc_cache_tx* tx,
                            uint64_t n, uint64_t ts_base, orc_cache_result* results, orc_entry* log);
void orc_gen_cache_batch(uint64_t seed, uint64_t n, uint64_t key_space, double alpha, uint32_t get_permille,
                         int32_t part, uint32_t steal_permille, orc_cache_tx* out);
void orc_zipf_fill(uint64_t seed, uint64_t n, uint64_t span, double alpha, uint64_t* out);
void orc_gen_host_log(uint64_t seed, uint64_t n_tx, uint32_t writes_per_tx, uint32_t n_threads,
                      uint64_t lo, uint64_t span, uint64_t ts_base, orc_entry* out);

/* ---- CPU baselines: the reference CPU path on T host threads ----
 * guest-stm-batch worker pool with per-word versioned locks.
 * Returns committed count; tickets_out (nullable) gets commit tickets. */
uint64_t orc_mt_bank_batch(uint64_t* stmr, uint64_t base, uint64_t size_words, const orc_bank_tx* tx,
                           uint64_t n, int threads, uint64_t lock_entries, uint64_t* tickets_out,
                           uint64_t* rs, uint64_t* ws, uint64_t* chunks, uint64_t gran_bytes,
                           uint64_t chunk_bytes);
/* validateChunk(apply) on T threads over log partitions with the TS lock bit
 * (SPEC.md:348). */
int orc_mt_validate_apply(const orc_entry* e, uint64_t n, const uint64_t* rs_words, uint64_t gran_bytes,
                          uint64_t base, uint64_t* ts, uint64_t* dev, int threads, int apply);

/* ---- checker: P1 / P2-dagger over execution traces,
 * checker.c.  orc_trace_event mirrors capi.h hetm_trace_event (40 B). */
typedef struct {
    uint64_t seq, tx, addr, value;
    uint32_t round;
    uint8_t device, kind;
    uint16_t pad;
} orc_trace_event;
enum { ORC_CHECK_PASS = 0, ORC_CHECK_FAIL = 1, ORC_CHECK_INCOMPLETE = 2 };
enum { ORC_REASON_NONE = 0, ORC_REASON_READ = 1, ORC_REASON_REALTIME = 2, ORC_REASON_INCOMPLETE = 3,
       ORC_REASON_BAD_ADDR = 4 };
typedef struct {
    int verdict, reason;
    uint64_t tx, addr, expected, got; /* witness: first inconsistent read (or real-time pair bound / ts) */
    uint32_t round;
    uint64_t checked_txs, checked_reads;
} orc_check_result;
/* P1: the finally committed transactions explained by the claimed serial order
 * (per round: host by commit ts, then device by ticket) from `init`. */
int orc_check_p1(const orc_trace_event* ev, uint64_t n, const uint64_t* init, uint64_t words, orc_check_result* res);
/* P2-dagger: every speculatively committed transaction of an aborted side
 * explained by the committed state plus its own device's speculative set. */
int orc_check_p2dagger(const orc_trace_event* ev, uint64_t n, const uint64_t* init, uint64_t words,
                       orc_check_result* res);

#ifdef __cplusplus
}
#endif
#endif
