// phased_tx.cuh — warp-phased PR-STM commit for transactions whose read and
// write sets are known at begin (bank transfers: the read set is the input).
//
// Same lock protocol as device_tm.cuh (64-bit versioned locks, priority
// pre-locks that a higher priority may steal, FINAL lock during write-back,
// commit ticket taken after the write claims are visible and before the read
// set is validated), reorganised so a warp walks the phases in lock-step and
// every phase issues its memory operations back to back:
//
//   P1  lock words of the NR read addresses                      (1 round trip)
//   P2  STMR loads  ||  pre-lock CAS of the NW write entries     (1 round trip)
//   P3  one ticket atomicAdd per warp for the surviving lanes    (1 round trip)
//   P4  validation loads of read-only entries || finalize CAS    (1 round trip)
//   P5  write back, fence, release, bitmap REDs                  (1 round trip)
//
// Data loads may be issued before the pre-lock CAS completes: any writer that
// touched a word between P1 and our CAS changed its lock word, so the CAS
// (which expects the P1 value) fails and the attempt is retried.  The data
// loads themselves are control-dependent on the P1 lock words (no FINAL seen).
#pragma once
#include "device_tm.cuh"

namespace hetm_b200 {

// RED-if-unset: a weak (L1-cacheable) probe first; bits only accrete within a
// round, so a stale 0 just costs a redundant RED.
__device__ __forceinline__ void set_bit_probe(unsigned long long* words, uint64_t bit) {
    const unsigned long long m = 1ull << (bit & 63);
    if (!(words[bit >> 6] & m)) atomicOr(&words[bit >> 6], m);
}

template <int NR, int NW>
struct StaticTx {
    uint64_t loc[NR];      // local word index of read k (writes are reads 0..NW-1)
    uint32_t lk[NR];       // lock index of read k
    unsigned long long l[NR];  // lock word seen in P1
    uint64_t val[NR];      // value read
    uint64_t wval[NW];     // value to write to loc[j], j < NW
};

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

// One phased attempt for every lane with `active`; returns true on commit and
// sets `ticket`.  All 32 lanes of the warp must call it together.
// Knock-out bits for profiling experiments only (HETM_KNOCKOUT env var; 0 in
// production): they remove protocol steps and break serializability.
enum : int { KO_TICKET = 1, KO_FENCE = 2, KO_BITMAPS = 4, KO_FINALIZE = 8, KO_PRELOCK = 16, KO_LOCKLOAD = 32 };

template <int NR, int NW, int KO = 0, class Compute>
__device__ __forceinline__ bool phased_attempt(StaticTx<NR, NW>& tx, bool active, uint32_t me, const ShardView& v,
                                               const LockTable& lt, unsigned long long* ticket_ctr,
                                               unsigned long long& ticket, Compute compute) {
    bool ok = active;
    // ---- P1: lock words
    if (ok) {
#pragma unroll
        for (int k = 0; k < NR; ++k) tx.l[k] = (KO & KO_LOCKLOAD) ? 0ull : ld_relaxed(&lt.words[tx.lk[k]]);
#pragma unroll
        for (int k = 0; k < NR; ++k) {
            ok &= !(tx.l[k] & kLockFinal);
#pragma unroll
            for (int q = 0; q < k; ++q) ok &= !(tx.lk[q] == tx.lk[k] && tx.l[q] != tx.l[k]);
        }
#pragma unroll
        for (int j = 0; j < NW; ++j) {  // write entries: a higher-priority claim makes us back off
            const uint32_t own = lk_owner(tx.l[j]);
            ok &= (own == 0 || own > me);
        }
    }
    // ---- P2: data loads || pre-lock CAS (dedup write lock indices)
    bool held[NW];
#pragma unroll
    for (int j = 0; j < NW; ++j) held[j] = false;
    if (ok) {
#pragma unroll
        for (int k = 0; k < NR; ++k) tx.val[k] = ld_relaxed(&v.stmr[tx.loc[k]]);
        unsigned long long prev[NW];
#pragma unroll
        for (int j = 0; j < NW; ++j) {
            bool dup = false;
#pragma unroll
            for (int q = 0; q < j; ++q) dup |= (tx.lk[q] == tx.lk[j]);
            prev[j] = (dup || (KO & KO_PRELOCK)) ? tx.l[j]
                                                 : atomicCAS(&lt.words[tx.lk[j]], tx.l[j], lk_make(me, lk_ver(tx.l[j])));
            if (KO & KO_PRELOCK) dup = false;
            held[j] = !dup && prev[j] == tx.l[j];
            ok &= dup || held[j];
        }
        if (!ok) {
#pragma unroll
            for (int j = 0; j < NW; ++j)
                if (held[j]) atomicCAS(&lt.words[tx.lk[j]], lk_make(me, lk_ver(tx.l[j])), lk_make(0, lk_ver(tx.l[j])));
        }
    }
    // ---- P3: ticket (after every surviving lane's claims are performed)
    const unsigned long long t = (KO & KO_TICKET) ? (unsigned long long)me : warp_ticket(ok, ticket_ctr);
    // ---- P4: validate read-only entries || finalize write entries
    bool fin[NW];
#pragma unroll
    for (int j = 0; j < NW; ++j) fin[j] = false;
    uint32_t stolen_mask = 0;
    if (ok) {
        unsigned long long cur[NR];
        bool check[NR];
#pragma unroll
        for (int k = NW; k < NR; ++k) {
            bool mine = false;
#pragma unroll
            for (int q = 0; q < k; ++q) mine |= (tx.lk[q] == tx.lk[k]);
            check[k] = !mine;
            if (check[k]) cur[k] = ld_relaxed(&lt.words[tx.lk[k]]);
        }
        unsigned long long fprev[NW];
#pragma unroll
        for (int j = 0; j < NW; ++j) {
            const unsigned long long exp = lk_make(me, lk_ver(tx.l[j]));
            if (held[j]) {
                fprev[j] = (KO & KO_FINALIZE) ? exp : atomicCAS(&lt.words[tx.lk[j]], exp, exp | kLockFinal);
                fin[j] = fprev[j] == exp;
                ok &= fin[j];
            }
        }
#pragma unroll
        for (int k = NW; k < NR; ++k) {
            if (!check[k] || !ok) continue;
            unsigned long long c = cur[k];
            for (;;) {  // rare loop: steal a lower-priority pre-lock on a read entry
                if ((c & kLockFinal) || lk_ver(c) != lk_ver(tx.l[k])) { ok = false; break; }
                const uint32_t own = lk_owner(c);
                if (own == 0 || own == me) break;
                if (own < me) { ok = false; break; }
                const unsigned long long p = atomicCAS(&lt.words[tx.lk[k]], c, lk_make(me, lk_ver(tx.l[k])));
                if (p == c) { stolen_mask |= 1u << k; break; }
                c = p;
            }
        }
    }
    if (active && !ok) {  // unwind whatever this attempt still holds
#pragma unroll
        for (int j = 0; j < NW; ++j) {
            const unsigned long long plain = lk_make(0, lk_ver(tx.l[j]));
            if (fin[j]) st_relaxed(&lt.words[tx.lk[j]], plain);
            else if (held[j]) atomicCAS(&lt.words[tx.lk[j]], lk_make(me, lk_ver(tx.l[j])), plain);
        }
#pragma unroll
        for (int k = NW; k < NR; ++k)
            if (stolen_mask & (1u << k))
                atomicCAS(&lt.words[tx.lk[k]], lk_make(me, lk_ver(tx.l[k])), lk_make(0, lk_ver(tx.l[k])));
        return false;
    }
    if (!ok) return false;
    // ---- P5: write back, release, instrument
    compute(tx);
#pragma unroll
    for (int j = 0; j < NW; ++j) st_relaxed(&v.stmr[tx.loc[j]], tx.wval[j]);
    if (!(KO & KO_FENCE)) fence_acq_rel();
    const uint32_t nv = (uint32_t)(t + 1);
#pragma unroll
    for (int j = 0; j < NW; ++j)
        if (fin[j]) st_relaxed(&lt.words[tx.lk[j]], lk_make(0, nv));
#pragma unroll
    for (int k = NW; k < NR; ++k)
        if (stolen_mask & (1u << k))
            atomicCAS(&lt.words[tx.lk[k]], lk_make(me, lk_ver(tx.l[k])), lk_make(0, lk_ver(tx.l[k])));
    // fire-and-forget REDs: they drain while the next attempt's loads are in flight
    if constexpr ((KO & KO_BITMAPS) == 0) {
#pragma unroll
        for (int k = 0; k < NR; ++k) set_bit(v.rs, tx.loc[k] >> v.gran_shift);
#pragma unroll
        for (int j = 0; j < NW; ++j) {
            set_bit(v.ws, tx.loc[j] >> v.gran_shift);
            set_bit(v.chunk, tx.loc[j] >> v.chunk_shift);
        }
    }
    ticket = t;
    return true;
}

}  // namespace hetm_b200
