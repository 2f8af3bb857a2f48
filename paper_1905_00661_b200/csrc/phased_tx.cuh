// phased_tx.cuh — warp-phased PR-STM commit for transactions whose read and
// write sets are known at begin (bank transfers: the read set is the input).
//
// Same lock protocol as device_tm.cuh (per-word versioned locks in the word
// cells, priority pre-locks that a higher priority may steal, FINAL lock during
// write-back, commit ticket taken after the write claims are visible and
// before the read set is validated), reorganised so a warp walks the phases in
// lock-step and every phase issues its memory operations back to back:
//
//   P1  128-bit {value, lock} snapshots of the NR words     (1 DRAM round trip)
//   P2  pre-lock CAS of the NW write words                   (L2 hit)
//       A CAS lost to a lower-priority claim is retried as a steal, so the
//       highest-priority transaction never loses a lock race.
//   P3  one ticket atomicAdd per warp for the surviving lanes
//   P4  validation loads of read-only words || finalize CAS  (L2 hits)
//       A read-only word held FINAL by a LOWER-priority transaction is waited
//       for (its holder only ever waits on still lower priorities, so waits
//       cannot cycle); a higher-priority claim aborts the attempt; a
//       lower-priority pre-lock is stolen.  Aborting on every FINAL instead
//       would let two transactions that read each other's write word abort
//       each other forever.
//   P5  128-bit {value, unlocked new version} stores + bitmap REDs (no wait)
//
// Writes are reads 0..NW-1 (no blind writes).  Duplicate words
// inside one transaction are handled: each distinct word is locked,
// validated and stored once (the last write to it wins, as in the oracle's
// sequential replay).
#pragma once
#include "device_tm.cuh"

namespace hetm_b200 {

template <int NR, int NW>
struct StaticTx {
    uint64_t loc[NR];          // local word index of read k (writes are reads 0..NW-1)
    unsigned long long l[NR];  // lock word seen in P1
    uint64_t val[NR];          // value read in P1
    uint64_t wval[NW];         // value to write to loc[j], j < NW
    uint32_t first;            // bit k set: loc[k] is the first occurrence of its word
};

template <int NR>
__device__ __forceinline__ uint32_t first_occurrences(const uint64_t (&loc)[NR]) {
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

// Knock-out bits for profiling experiments only (HETM_KNOCKOUT env var; 0 in
// production): they remove protocol steps and break serializability.
enum : int { KO_TICKET = 1, KO_BITMAPS = 4, KO_FINALIZE = 8 };

// One phased attempt for every lane with `active`; returns true on commit and
// sets `ticket`.  All 32 lanes of the warp must call it together.
template <int NR, int NW, int KO = 0, class Compute>
__device__ __forceinline__ bool phased_attempt(StaticTx<NR, NW>& tx, bool active, uint32_t me, const ShardView& v,
                                               unsigned long long* ticket_ctr, unsigned long long& ticket,
                                               Compute compute) {
    bool ok = active;
    // ---- P1: consistent {value, lock} snapshots
    if (ok) {
#pragma unroll
        for (int k = 0; k < NR; ++k) ld_pair(&v.cells[tx.loc[k]], tx.val[k], tx.l[k]);
#pragma unroll
        for (int k = 0; k < NR; ++k) {
            ok &= !(tx.l[k] & kLockFinal);
#pragma unroll
            for (int q = 0; q < k; ++q)  // a word snapshotted twice must agree
                ok &= !(tx.loc[q] == tx.loc[k] && (tx.l[q] != tx.l[k] || tx.val[q] != tx.val[k]));
        }
#pragma unroll
        for (int j = 0; j < NW; ++j) {  // write words: a higher-priority claim makes us back off
            const uint32_t own = lk_owner(tx.l[j]);
            ok &= (own == 0 || own > me);
        }
    }
    // ---- P2: pre-lock CAS of the distinct write words
    bool held[NW];
#pragma unroll
    for (int j = 0; j < NW; ++j) held[j] = false;
    if (ok) {
        unsigned long long prev[NW];
#pragma unroll
        for (int j = 0; j < NW; ++j)
            if (tx.first & (1u << j))
                prev[j] = atomicCAS(&v.cells[tx.loc[j]].lock, tx.l[j], lk_make(me, lk_ver(tx.l[j])));
#pragma unroll
        for (int j = 0; j < NW; ++j) {
            if (!(tx.first & (1u << j))) continue;
            unsigned long long c = prev[j];
            const unsigned long long mine = lk_make(me, lk_ver(tx.l[j]));
            bool got = c == tx.l[j];
            // Lost the race: steal from a lower-priority pre-lock holder (possibly a
            // lane of this very warp), back off from a higher one (rare path).
            while (!got) {
                const uint32_t own = lk_owner(c);
                if ((c & kLockFinal) || lk_ver(c) != lk_ver(tx.l[j]) || (own != 0 && own < me)) break;
                const unsigned long long expect = c;
                c = atomicCAS(&v.cells[tx.loc[j]].lock, expect, mine);
                got = c == expect;
            }
            held[j] = got;
            ok &= got;
        }
        if (!ok) {
#pragma unroll
            for (int j = 0; j < NW; ++j)
                if (held[j])
                    atomicCAS(&v.cells[tx.loc[j]].lock, lk_make(me, lk_ver(tx.l[j])), lk_make(0, lk_ver(tx.l[j])));
        }
    }
    // ---- P3: ticket (after every surviving lane's claims are performed)
    const unsigned long long t = (KO & KO_TICKET) ? (unsigned long long)me : warp_ticket(ok, ticket_ctr);
    // ---- P4: validate read-only words || finalize write words
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
            for (int q = 0; q < NW; ++q) mine |= (tx.loc[q] == tx.loc[k]);
            check[k] = !mine && (tx.first & (1u << k));
            if (check[k]) cur[k] = ld_relaxed(&v.cells[tx.loc[k]].lock);
        }
        unsigned long long fprev[NW];
#pragma unroll
        for (int j = 0; j < NW; ++j) {
            const unsigned long long exp = lk_make(me, lk_ver(tx.l[j]));
            if (held[j])
                fprev[j] = (KO & KO_FINALIZE) ? exp : atomicCAS(&v.cells[tx.loc[j]].lock, exp, exp | kLockFinal);
        }
#pragma unroll
        for (int j = 0; j < NW; ++j)
            if (held[j]) {
                fin[j] = fprev[j] == lk_make(me, lk_ver(tx.l[j]));
                ok &= fin[j];
            }
#pragma unroll
        for (int k = NW; k < NR; ++k) {
            if (!check[k] || !ok) continue;
            unsigned long long c = cur[k];
            for (;;) {  // rare loop: priority rule on a claimed read-only word
                if (lk_ver(c) != lk_ver(tx.l[k])) { ok = false; break; }  // someone committed it
                const uint32_t own = lk_owner(c);
                if (own != 0 && own < me) { ok = false; break; }          // higher priority claims it
                if (c & kLockFinal) {  // lower-priority holder mid-commit: wait for its release
                    c = ld_relaxed(&v.cells[tx.loc[k]].lock);
                    continue;
                }
                if (own == 0 || own == me) break;
                const unsigned long long p = atomicCAS(&v.cells[tx.loc[k]].lock, c, lk_make(me, lk_ver(tx.l[k])));
                if (p == c) { stolen_mask |= 1u << k; break; }
                c = p;
            }
        }
    }
    if (active && !ok) {  // unwind whatever this attempt still holds
#pragma unroll
        for (int j = 0; j < NW; ++j) {
            const unsigned long long plain = lk_make(0, lk_ver(tx.l[j]));
            if (fin[j]) st_relaxed(&v.cells[tx.loc[j]].lock, plain);
            else if (held[j]) atomicCAS(&v.cells[tx.loc[j]].lock, lk_make(me, lk_ver(tx.l[j])), plain);
        }
#pragma unroll
        for (int k = NW; k < NR; ++k)
            if (stolen_mask & (1u << k))
                atomicCAS(&v.cells[tx.loc[k]].lock, lk_make(me, lk_ver(tx.l[k])), lk_make(0, lk_ver(tx.l[k])));
        return false;
    }
    if (!ok) return false;
    // ---- P5: write back + release in one 128-bit store per distinct written word
    compute(tx);
    const uint32_t nv = (uint32_t)(t + 1);
#pragma unroll
    for (int j = 0; j < NW; ++j) {
        if (!held[j]) continue;
        uint64_t val = tx.wval[j];
#pragma unroll
        for (int q = j + 1; q < NW; ++q)
            if (tx.loc[q] == tx.loc[j]) val = tx.wval[q];  // the last write to a word wins
        st_pair(&v.cells[tx.loc[j]], val, lk_make(0, nv));
    }
#pragma unroll
    for (int k = NW; k < NR; ++k)
        if (stolen_mask & (1u << k))
            atomicCAS(&v.cells[tx.loc[k]].lock, lk_make(me, lk_ver(tx.l[k])), lk_make(0, lk_ver(tx.l[k])));
    // fire-and-forget REDs: they drain while the next attempt's loads are in flight
    if constexpr ((KO & KO_BITMAPS) == 0) {
#pragma unroll
        for (int k = 0; k < NR; ++k)
            if (tx.first & (1u << k)) set_bit(v.rs, tx.loc[k] >> v.gran_shift);
#pragma unroll
        for (int j = 0; j < NW; ++j)
            if (held[j]) {
                set_bit(v.ws, tx.loc[j] >> v.gran_shift);
                set_bit(v.chunk, tx.loc[j] >> v.chunk_shift);
            }
    }
    ticket = t;
    return true;
}

}  // namespace hetm_b200
