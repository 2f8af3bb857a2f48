// phased_tx.cuh — warp-phased commit for transactions whose read and write
// sets are known at begin (bank transfers: the read set is the input).
//
// Same lock word and serial order as device_tm.cuh (per-word versioned locks
// in the word cells; commit ticket taken after the write locks are visible
// and before the read set is validated), reorganised so a warp walks the
// phases in lock-step and every phase issues its memory operations back to
// back.  Write words are locked straight to FINAL (commit-time locking): a
// batch-phase transaction holds its locks only for its own short commit
// window, so the pre-lock/steal stage of device_tm.cuh — one extra atomic per
// written word — is replaced by priority-ordered WAITING:
//
//   P1  128-bit {value, lock} snapshot of each written word, lock word of each
//       read-only word, weak probes of the RS/WS/ChunkMap words (1 DRAM trip)
//   P2  CAS unlocked(version) -> FINAL|prio|version on the written words; a
//       lost race against a LOWER-priority holder waits for its release and
//       retries, a higher-priority holder or a new version aborts
//   P3  one ticket atomicAdd per group of converged surviving lanes
//   P4  validation loads of the read-only words.  Priority rule: a word held
//       FINAL by a LOWER-priority transaction is waited for (that holder only
//       ever waits on still lower priorities, so waits cannot cycle and the
//       highest-priority live transaction never waits); a higher-priority
//       holder or a changed version aborts the attempt.
//   P5  128-bit {value, unlocked new version} store per written word (write
//       back and release in one access), REDs only for bitmap bits the P1
//       probe found clear (bits accrete within a round, so a stale clear probe
//       only costs a redundant RED).
//
// Duplicate words inside one transaction are handled: each distinct word is
// locked, validated and stored once (the last write to it wins, as in the
// oracle's sequential replay).
//
// KO_STRIPES (the product bank kernel): the versioned lock words live in an
// L2-resident STRIPE TABLE (ShardView::stripes, 2^24 32-bit words = 64 MiB, word ->
// stripe by a multiplicative hash) instead of the cells' meta words.  Only the
// written cells are then touched in DRAM (one 128-bit load, one 128-bit
// store); every lock/validation access is an L2 hit
// (tools/stripe_probe.cu: 0.152 vs 0.275 ms for the same access shape,
// profiles/r02l_stripe_probe.txt).  The phases become
//   P0  stripe words of all accounts + bitmap probes (one L2 round trip)
//   P2  CAS on the distinct written stripes
//   P1  128-bit {value, meta} of the written cells, issued once the CAS
//       returned (control dependency, the ordering argument of the ticket ->
//       validation step of device_tm.cuh): the cells are read under the
//       locks, and their DRAM round trip overlaps P3/P4 instead of preceding
//       the locks
//   P3  ticket; P4 reload of the read-only stripes not held by this transaction
//   P5  128-bit {value, lk_commit(ticket)} per written cell (the cell keeps
//       its last writer's version for the merge pick pass), fence.release.gpu,
//       release of the held stripes with the same version.
// Distinct words sharing a stripe are locked / validated once (false sharing
// only costs an occasional abort).  Kernels that lock the cells' meta words
// (rw, cache, device_tm.cuh) never run concurrently with a bank batch: batches
// are serialised on the execution stream.
#pragma once
#include "device_tm.cuh"

namespace hetm_b200 {

// Words 0..NW-1 are read-modify-written (their values are snapshotted with the
// lock, 128-bit); words NW..NR-1 are read-only and only their lock word is
// loaded (bank: accounts 2 and 3 are read for validation, their values unused).
template <int NR, int NW>
struct StaticTx {
    uint32_t loc[NR];          // local word (cell) index; shards hold < 2^32 words
    unsigned long long l[NR];  // lock word seen in P1
    uint64_t val[NW];          // value of write word j seen in P1
    uint64_t wval[NW];         // value to write to loc[j]
    uint64_t rv[NR > NW ? NR - NW : 1];  // KO_TRACE only: value of read-only word NW+k seen in P1
    uint32_t first;            // bit k set: loc[k] is the first occurrence of its word
    uint32_t block_loc;        // abort cause: lock word (cell, or stripe under KO_STRIPES) held FINAL ...
    unsigned long long block_lk;  // ... with this value (0: no such blocker)
    uint32_t sidx[NR];         // KO_STRIPES: stripe of loc[k]
    uint32_t sfirst;           // KO_STRIPES: bit k set: sidx[k] is the first occurrence of its stripe
};

// Stripe of a local word (KO_STRIPES): Fibonacci hash, so neighbouring (hot,
// zipf-ranked) accounts land on different stripes.
__device__ __forceinline__ uint32_t stripe_of(uint32_t loc, uint32_t stripe_shift) {
    return (uint32_t)(((uint64_t)loc * 0x9e3779b97f4a7c15ull) >> stripe_shift);
}

template <int NR>
__device__ __forceinline__ uint32_t first_occurrences(const uint32_t (&loc)[NR]) {
    uint32_t m = 0;
#pragma unroll
    for (int k = 0; k < NR; ++k) {
        bool seen = false;
#pragma unroll
        for (int q = 0; q < k; ++q) seen |= (loc[q] == loc[k]);
        if (!seen) m |= 1u << k;
    }
    return m;
}

// Warp-aggregated ticket over the lanes with `ok`; all 32 lanes must call.
__device__ __forceinline__ unsigned long long warp_ticket(bool ok, unsigned long long* ctr) {
    const unsigned m = __ballot_sync(0xffffffffu, ok);
    unsigned long long base = 0;
    if (m) {
        const unsigned leader = __ffs(m) - 1;
        if (lane_id() == leader) base = atomicAdd(ctr, (unsigned long long)__popc(m));
        base = __shfl_sync(0xffffffffu, base, leader);
    }
    return base + __popc(m & ((1u << lane_id()) - 1u));
}

// Diagnostics only (HETM_KNOCKOUT env var, 0 in production): KO_PROTOCOL
// keeps the snapshot loads and stores and drops every protocol step (the
// access-pattern floor); KO_PHASE_CLOCKS accumulates per-phase cycles.
// KO_COUNT_TICKETS counts ticket atomics (debug word 4).
enum : int {
    KO_BITMAPS = 4, KO_NO_PROBE = 8, KO_COUNT_TICKETS = 16, KO_PROTOCOL = 64,
    KO_PHASE_CLOCKS = 128, KO_LOCK_READS = 256, KO_SKIP_VALIDATE = 512, KO_NO_TICKET = 1024,
    KO_TRACE = 2048,  // checker traces: also load the VALUES of the read-only words (tx.rv)
    KO_STRIPES = 4096,  // lock words in the L2-resident stripe table (product bank kernel)
    KO_STRIPE_SPIN = 8192,  // KO_STRIPES: a stripe found locked in P0 is waited for (bounded) instead of aborting
    KO_NO_FENCE = 16384,    // KO_STRIPES knockout (experiments only, INCORRECT): no release fence
    KO_STRIPE_2PL = 32768   // KO_STRIPES: lock the read-only stripes too (no validation phase)
};

// Stripe words (KO_STRIPES) are 32 bits: unlocked = the 31-bit commit version
// of the stripe's last writer (lk_commit), locked = kStripeFinal | owner
// priority.  A locked stripe hides its version; a waiter compares it after
// the release, so the priority rule and the abort decisions are unchanged
// (a holder on a changed version is waited for, then the change aborts).
constexpr unsigned int kStripeFinal = 0x80000000u;
__device__ __forceinline__ unsigned int stripe_lock(uint32_t me) { return kStripeFinal | me; }
__device__ __forceinline__ uint32_t stripe_owner(unsigned int c) { return c & ~kStripeFinal; }

// Current value of the lock word guarding lock index `idx` (a cell index, or a
// stripe index under KO_STRIPES), widened to 64 bits for the sit-out poll.
template <int KO>
__device__ __forceinline__ unsigned long long lock_value(const ShardView& v, uint32_t idx) {
    if constexpr ((KO & KO_STRIPES) != 0) return ld_relaxed(&v.stripes[idx]);
    else return ld_relaxed(&v.cells[idx].meta);
}

__device__ __forceinline__ void phase_mark(unsigned long long* acc, int phase, long long& t) {
    const long long now = clock64();
    acc[phase] += (unsigned long long)(now - t);
    if (phase == 0) acc[5] += 1;
    t = now;
}

// One phased attempt for every lane with `active`; returns true on commit and
// sets `ticket`.  An attempt that took a ticket and then aborted also reports
// it (its write-set log slots must be cleared); otherwise ticket = ~0.  All
// 32 lanes of the warp must call it together.
template <int NR, int NW, int KO = 0, class Compute>
__device__ __forceinline__ bool phased_attempt(StaticTx<NR, NW>& tx, bool active, uint32_t me, const ShardView& v,
                                               unsigned long long* ticket_ctr, unsigned long long& ticket,
                                               Compute compute, unsigned long long* clocks = nullptr) {
    bool ok = active;
    if (active) tx.block_lk = 0;  // a sitting-out lane keeps its blocker
    long long tclk = 0;
    if constexpr ((KO & KO_PHASE_CLOCKS) != 0) tclk = clock64();
    if constexpr ((KO & KO_PROTOCOL) != 0) {  // access-pattern floor
        if (!ok) return false;
#pragma unroll
        for (int k = 0; k < NR; ++k) {
            if (k < NW) ld_pair(&v.cells[tx.loc[k]], tx.val[k < NW ? k : 0], tx.l[k]);
            else tx.l[k] = ld_relaxed(&v.cells[tx.loc[k]].meta);
        }
        compute(tx);
#pragma unroll
        for (int j = 0; j < NW; ++j) st_pair(&v.cells[tx.loc[j]], tx.wval[j], tx.l[j]);
        ticket = me;
        return true;
    }
    // ---- P1: snapshots + bitmap probes
    uint32_t need_bits = 0;  // bit k: RS bit of word k clear; bit NR+j: WS, bit NR+NW+j: chunk
    if (ok) {
#pragma unroll
        for (int k = 0; k < NR; ++k) {
            if (k < NW) ld_pair(&v.cells[tx.loc[k]], tx.val[k < NW ? k : 0], tx.l[k]);
            else if constexpr ((KO & KO_TRACE) != 0) ld_pair(&v.cells[tx.loc[k]], tx.rv[k >= NW ? k - NW : 0], tx.l[k]);
            else tx.l[k] = ld_relaxed(&v.cells[tx.loc[k]].meta);
        }
        unsigned long long pr[NR + 2 * NW];
        if constexpr ((KO & (KO_NO_PROBE | KO_BITMAPS)) != 0) {
#pragma unroll
            for (int k = 0; k < NR + 2 * NW; ++k) pr[k] = (KO & KO_BITMAPS) ? ~0ull : 0ull;
        } else {
#pragma unroll
            for (int k = 0; k < NR; ++k) pr[k] = v.rs[(tx.loc[k] >> v.gran_shift) >> 6];
#pragma unroll
            for (int j = 0; j < NW; ++j) {
                pr[NR + j] = v.ws[(tx.loc[j] >> v.gran_shift) >> 6];
                pr[NR + NW + j] = v.chunk[(tx.loc[j] >> v.chunk_shift) >> 6];
            }
        }
#pragma unroll
        for (int k = 0; k < NR; ++k) {
            if (tx.l[k] & kLockFinal) {
                ok = false;
                tx.block_loc = tx.loc[k];
                tx.block_lk = tx.l[k];
            }
            // a word loaded twice must show one lock word (values only change
            // together with the version, so equal unlocked lock words imply equal values)
#pragma unroll
            for (int q = 0; q < k; ++q) ok &= !(tx.loc[q] == tx.loc[k] && tx.l[q] != tx.l[k]);
            if (!((pr[k] >> ((tx.loc[k] >> v.gran_shift) & 63)) & 1ull)) need_bits |= 1u << k;
        }
#pragma unroll
        for (int j = 0; j < NW; ++j) {
            if (!((pr[NR + j] >> ((tx.loc[j] >> v.gran_shift) & 63)) & 1ull)) need_bits |= 1u << (NR + j);
            if (!((pr[NR + NW + j] >> ((tx.loc[j] >> v.chunk_shift) & 63)) & 1ull))
                need_bits |= 1u << (NR + NW + j);
        }
    }
    if constexpr ((KO & KO_PHASE_CLOCKS) != 0) phase_mark(clocks, 0, tclk);
    // ---- P2: lock the distinct written words (unlocked version -> FINAL);
    // with kLockReads the read-only words too (2PL: no validation phase)
    constexpr bool kLockReads = (KO & KO_LOCK_READS) != 0;
    constexpr int NL = kLockReads ? NR : NW;  // words locked in P2
    bool held[NL];
#pragma unroll
    for (int j = 0; j < NL; ++j) held[j] = false;
    if (ok) {
        unsigned long long prev[NL];
#pragma unroll
        for (int j = 0; j < NL; ++j)
            if (tx.first & (1u << j))
                prev[j] = atomicCAS(&v.cells[tx.loc[j]].meta, tx.l[j], kLockFinal | lk_make(me, lk_ver(tx.l[j])));
#pragma unroll
        for (int j = 0; j < NL; ++j) held[j] = (tx.first & (1u << j)) && prev[j] == tx.l[j];
#pragma unroll
        for (int j = 0; j < NL; ++j) {
            if (!(tx.first & (1u << j)) || held[j] || !ok) continue;
            unsigned long long c = prev[j];
            // Lost the race: wait for a LOWER-priority holder to commit or back
            // off, then retry; a higher-priority holder or a new version aborts.
            while (c != tx.l[j]) {
                if (lk_ver(c) != lk_ver(tx.l[j]) || !(c & kLockFinal) || lk_owner(c) < me) {
                    if ((c & kLockFinal) && lk_ver(c) == lk_ver(tx.l[j])) {
                        tx.block_loc = tx.loc[j];
                        tx.block_lk = c;
                    }
                    ok = false;
                    break;
                }
                c = ld_relaxed(&v.cells[tx.loc[j]].meta);
                if (c == tx.l[j])
                    c = atomicCAS(&v.cells[tx.loc[j]].meta, tx.l[j], kLockFinal | lk_make(me, lk_ver(tx.l[j])));
            }
            held[j] = c == tx.l[j];
        }
        if (!ok) {
#pragma unroll
            for (int j = 0; j < NL; ++j)
                if (held[j]) st_relaxed(&v.cells[tx.loc[j]].meta, tx.l[j]);  // nothing written: restore
        }
    }
    if constexpr ((KO & KO_PHASE_CLOCKS) != 0) phase_mark(clocks, 1, tclk);
    // ---- P3: ticket (after every surviving lane's locks are performed).  Only
    // the converged surviving lanes aggregate: a lane may still be waiting on
    // a lower-priority holder of this very warp, so no full-warp collective
    // may separate lock acquisition from release.
    unsigned long long t = ~0ull;  // no ticket
    if constexpr ((KO & KO_NO_TICKET) != 0) {
        if (ok) t = me;
    } else {
        if (ok) t = take_ticket(ticket_ctr);
    }
    if constexpr ((KO & KO_COUNT_TICKETS) != 0) {
        if (ok && lane_id() == (unsigned)(__ffs(__activemask()) - 1)) clocks[0] += 1;
    }
    if constexpr ((KO & KO_PHASE_CLOCKS) != 0) phase_mark(clocks, 2, tclk);
    // ---- P4: validate the read-only words (not needed when they are locked)
    if (!kLockReads && (KO & KO_SKIP_VALIDATE) == 0 && ok) {
        unsigned long long cur[NR];
        bool check[NR];
#pragma unroll
        for (int k = NW; k < NR; ++k) {
            bool mine = false;
#pragma unroll
            for (int q = 0; q < NW; ++q) mine |= (tx.loc[q] == tx.loc[k]);
            check[k] = !mine && (tx.first & (1u << k));
            if (check[k]) cur[k] = ld_relaxed(&v.cells[tx.loc[k]].meta);
        }
#pragma unroll
        for (int k = NW; k < NR; ++k) {
            if (!check[k]) continue;
            unsigned long long c = cur[k];
            while (ok) {
                if (lk_ver(c) != lk_ver(tx.l[k])) ok = false;                 // committed since P1
                else if (!(c & kLockFinal)) break;                            // unclaimed: valid
                else if (lk_owner(c) < me) {                                  // higher priority holds it
                    ok = false;
                    tx.block_loc = tx.loc[k];
                    tx.block_lk = c;
                }
                else c = ld_relaxed(&v.cells[tx.loc[k]].meta);                // lower priority: wait
            }
        }
        if (!ok) {
#pragma unroll
            for (int j = 0; j < NL; ++j)
                if (held[j]) st_relaxed(&v.cells[tx.loc[j]].meta, tx.l[j]);
        }
    }
    if constexpr ((KO & KO_PHASE_CLOCKS) != 0) phase_mark(clocks, 3, tclk);
    if (!ok) {
        ticket = t;  // a ticket taken by an attempt that then aborted (0 = none taken)
        return false;
    }
    // ---- P5: write back + release in one 128-bit store per distinct written word
    compute(tx);
#pragma unroll
    for (int j = 0; j < NW; ++j) {
        if (!held[j]) continue;
        uint64_t val = tx.wval[j];
#pragma unroll
        for (int q = j + 1; q < NW; ++q)
            if (tx.loc[q] == tx.loc[j]) val = tx.wval[q];  // the last write to a word wins
        st_pair(&v.cells[tx.loc[j]], val, lk_commit(t));
    }
#pragma unroll
    for (int j = NW; j < NL; ++j)  // read-only words locked in P2: release, version unchanged
        if (held[j]) st_relaxed(&v.cells[tx.loc[j]].meta, tx.l[j]);
#pragma unroll
    for (int k = 0; k < NR; ++k)
        if ((need_bits >> k) & 1u) set_bit(v.rs, tx.loc[k] >> v.gran_shift);
#pragma unroll
    for (int j = 0; j < NW; ++j) {
        if ((need_bits >> (NR + j)) & 1u) set_bit(v.ws, tx.loc[j] >> v.gran_shift);
        if ((need_bits >> (NR + NW + j)) & 1u) set_bit(v.chunk, tx.loc[j] >> v.chunk_shift);
    }
    if constexpr ((KO & KO_PHASE_CLOCKS) != 0) phase_mark(clocks, 4, tclk);
    ticket = t;
    return true;
}

// KO_STRIPES form of phased_attempt (header comment): same contract, same
// priority rule and waiting discipline, lock words in the stripe table.
template <int NR, int NW, int KO, class Compute>
__device__ __forceinline__ bool striped_attempt(StaticTx<NR, NW>& tx, bool active, uint32_t me, const ShardView& v,
                                                unsigned long long* ticket_ctr, unsigned long long& ticket,
                                                Compute compute) {
    static_assert((KO & (KO_PROTOCOL | KO_LOCK_READS | KO_PHASE_CLOCKS)) == 0, "cell-lock experiments only");
    bool ok = active;
    if (active) tx.block_lk = 0;
    unsigned int sl[NR];        // stripe words seen in P0
    uint32_t need_bits = 0;     // bit k: RS bit of word k clear; bit NR+j: WS, bit NR+NW+j: chunk
    // ---- P0: stripe words + bitmap probes (L2 hits, one round trip)
    if (ok) {
#pragma unroll
        for (int k = 0; k < NR; ++k)
            if (tx.sfirst & (1u << k)) sl[k] = ld_relaxed(&v.stripes[tx.sidx[k]]);
        unsigned long long pr[NR + 2 * NW];  // bitmap probes, in the same round trip
        if constexpr ((KO & (KO_NO_PROBE | KO_BITMAPS)) != 0) {  // knockouts (experiments only)
#pragma unroll
            for (int k = 0; k < NR + 2 * NW; ++k) pr[k] = (KO & KO_BITMAPS) ? ~0ull : 0ull;
        } else {
#pragma unroll
            for (int k = 0; k < NR; ++k) pr[k] = v.rs[(tx.loc[k] >> v.gran_shift) >> 6];
#pragma unroll
            for (int j = 0; j < NW; ++j) {
                pr[NR + j] = v.ws[(tx.loc[j] >> v.gran_shift) >> 6];
                pr[NR + NW + j] = v.chunk[(tx.loc[j] >> v.chunk_shift) >> 6];
            }
        }
#pragma unroll
        for (int k = 0; k < NR; ++k)
            if (!((pr[k] >> ((tx.loc[k] >> v.gran_shift) & 63)) & 1ull)) need_bits |= 1u << k;
#pragma unroll
        for (int j = 0; j < NW; ++j) {
            if (!((pr[NR + j] >> ((tx.loc[j] >> v.gran_shift) & 63)) & 1ull)) need_bits |= 1u << (NR + j);
            if (!((pr[NR + NW + j] >> ((tx.loc[j] >> v.chunk_shift) & 63)) & 1ull))
                need_bits |= 1u << (NR + NW + j);
        }
        if constexpr ((KO & KO_STRIPE_SPIN) != 0) {
            // no lock is held yet, so waiting here cannot close a cycle; a holder
            // is another warp mid-commit (a warp's own lanes hold nothing in P0)
#pragma unroll
            for (int k = 0; k < NR; ++k) {
                if (!(tx.sfirst & (1u << k))) continue;
                for (int p = 0; p < 64 && (sl[k] & kStripeFinal); ++p) {
                    __nanosleep(64);
                    sl[k] = ld_relaxed(&v.stripes[tx.sidx[k]]);
                }
            }
        }
#pragma unroll
        for (int k = 0; k < NR; ++k) {
            if (!(tx.sfirst & (1u << k))) {
#pragma unroll
                for (int q = 0; q < k; ++q)
                    if (tx.sidx[q] == tx.sidx[k] && (tx.sfirst & (1u << q))) sl[k] = sl[q];
            }
            if (sl[k] & kStripeFinal) {
                ok = false;
                tx.block_loc = tx.sidx[k];
                tx.block_lk = sl[k];
            }
        }
    }
        // ---- P2: lock the distinct written stripes (unlocked version -> FINAL);
    // with KO_STRIPE_2PL the read-only ones too
    constexpr int NL = (KO & KO_STRIPE_2PL) != 0 ? NR : NW;
    bool held[NL];
#pragma unroll
    for (int j = 0; j < NL; ++j) held[j] = false;
    if (ok) {
        unsigned int prev[NL];
#pragma unroll
        for (int j = 0; j < NL; ++j)
            if (tx.sfirst & (1u << j))
                prev[j] = atomicCAS(&v.stripes[tx.sidx[j]], sl[j], stripe_lock(me));
#pragma unroll
        for (int j = 0; j < NL; ++j) held[j] = (tx.sfirst & (1u << j)) && prev[j] == sl[j];
#pragma unroll
        for (int j = 0; j < NL; ++j) {
            if (!(tx.sfirst & (1u << j)) || held[j] || !ok) continue;
            unsigned int c = prev[j];
            while (c != sl[j]) {  // lost the race: wait for a LOWER-priority holder, else abort
                if (!(c & kStripeFinal) || stripe_owner(c) < me) {  // a new version, or a higher priority holds it
                    if (c & kStripeFinal) {
                        tx.block_loc = tx.sidx[j];
                        tx.block_lk = c;
                    }
                    ok = false;
                    break;
                }
                c = ld_relaxed(&v.stripes[tx.sidx[j]]);
                if (c == sl[j]) c = atomicCAS(&v.stripes[tx.sidx[j]], sl[j], stripe_lock(me));
            }
            held[j] = c == sl[j];
        }
        if (!ok) {
#pragma unroll
            for (int j = 0; j < NL; ++j)
                if (held[j]) st_relaxed(&v.stripes[tx.sidx[j]], sl[j]);  // nothing written: restore
        }
    }
    // ---- P1: the written cells, loaded UNDER the stripe locks (issued once the
    // CAS returned: control dependency), so their DRAM round trip overlaps the
    // ticket and the validation loads instead of preceding the locks; a held
    // stripe's last writer released it after a fence, so its value is visible
    if (ok) {
        unsigned long long meta;
#pragma unroll
        for (int k = 0; k < NR; ++k) {
            if (k < NW) ld_pair(&v.cells[tx.loc[k]], tx.val[k < NW ? k : 0], meta);
            else if constexpr ((KO & KO_TRACE) != 0) ld_pair(&v.cells[tx.loc[k]], tx.rv[k >= NW ? k - NW : 0], meta);
        }
    }
    // ---- P3: ticket (after every surviving lane's locks are performed)
    unsigned long long t = ~0ull;
    if constexpr ((KO & KO_NO_TICKET) != 0) {
        if (ok) t = me;
    } else {
        if (ok) t = take_ticket(ticket_ctr);
    }
    // ---- P4: validate the read-only stripes this transaction does not hold
    if ((KO & (KO_SKIP_VALIDATE | KO_STRIPE_2PL)) == 0 && ok) {
        unsigned int cur[NR];
        bool check[NR];
#pragma unroll
        for (int k = NW; k < NR; ++k) {
            bool mine = false;
#pragma unroll
            for (int q = 0; q < NW; ++q) mine |= (tx.sidx[q] == tx.sidx[k]);
            check[k] = !mine && (tx.sfirst & (1u << k));
            if (check[k]) cur[k] = ld_relaxed(&v.stripes[tx.sidx[k]]);
        }
#pragma unroll
        for (int k = NW; k < NR; ++k) {
            if (!check[k]) continue;
            unsigned int c = cur[k];
            while (ok) {
                if (!(c & kStripeFinal)) {                                    // unlocked: valid iff unchanged
                    ok = c == sl[k];
                    break;
                }
                if (stripe_owner(c) < me) {                                   // higher priority holds it
                    ok = false;
                    tx.block_loc = tx.sidx[k];
                    tx.block_lk = c;
                }
                else c = ld_relaxed(&v.stripes[tx.sidx[k]]);                  // lower priority: wait
            }
        }
        if (!ok) {
#pragma unroll
            for (int j = 0; j < NL; ++j)
                if (held[j]) st_relaxed(&v.stripes[tx.sidx[j]], sl[j]);
        }
    }
    if (!ok) {
        ticket = t;
        return false;
    }
    // ---- P5: write back the distinct written words, then release the stripes
    compute(tx);
    const unsigned long long ver = lk_commit(t);
    const unsigned int sver = (unsigned int)ver;  // 31-bit commit version, bit 31 clear
#pragma unroll
    for (int j = 0; j < NW; ++j) {
        if (!(tx.first & (1u << j))) continue;
        uint64_t val = tx.wval[j];
#pragma unroll
        for (int q = j + 1; q < NW; ++q)
            if (tx.loc[q] == tx.loc[j]) val = tx.wval[q];  // the last write to a word wins
        st_pair(&v.cells[tx.loc[j]], val, ver);
    }
    // release fence (MEMBAR without the L1 invalidate of fence.acq_rel): the cell
    // stores are performed before the stripe releases
    if constexpr ((KO & KO_NO_FENCE) == 0) asm volatile("fence.release.gpu;" ::: "memory");
#pragma unroll
    for (int j = 0; j < NL; ++j)  // written stripes publish the commit version, read-only ones keep theirs
        if (held[j]) st_relaxed(&v.stripes[tx.sidx[j]], j < NW ? sver : sl[j]);
    // bitmap bits after the releases, so the fence waits for the two cell
    // stores only; fire-and-forget REDs (explicit PTX: after a fence the
    // compiler emits returning ATOMs for atomicOr)
#pragma unroll
    for (int k = 0; k < NR; ++k)
        if ((need_bits >> k) & 1u) red_or_bit(v.rs, tx.loc[k] >> v.gran_shift);
#pragma unroll
    for (int j = 0; j < NW; ++j) {
        if ((need_bits >> (NR + j)) & 1u) red_or_bit(v.ws, tx.loc[j] >> v.gran_shift);
        if ((need_bits >> (NR + NW + j)) & 1u) red_or_bit(v.chunk, tx.loc[j] >> v.chunk_shift);
    }
    ticket = t;
    return true;
}

}  // namespace hetm_b200
