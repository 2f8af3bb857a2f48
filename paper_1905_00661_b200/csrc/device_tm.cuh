// device_tm.cuh — PR-STM-style device guest TM.
//
// Device-side TM_read / TM_write / TM_commit for transactional kernels.  One
// CUDA thread runs one transaction; every transaction eventually commits or
// reports livelock.
//
// Per-word versioned lock, the `meta` word of the word's cell (common.cuh):
//     bit 63      FINAL  — write-back in progress, never stolen
//     bits 61..32 owner  — priority of the pre-lock holder (0 = free)
//     bits 31..0  version — low 31 bits of the last committing ticket + 1
// A TS word (bit 62, left by validation) reads as an unlocked word of the
// reserved version 0xffffffff, which no commit produces (commit versions are
// 31-bit), so a value change is always a version change (no ABA).
// Priority rule (PR-STM): priority = batch index + 1, smaller wins.  A
// transaction may steal a lower-priority PRE-lock; the robbed transaction
// fails its finalize step and retries.  The highest-priority live transaction
// is therefore only ever aborted by a FINAL lock (its holder is already
// writing back) or by a version change (someone committed): no livelock.
//
// Commit (TL2 order, SURVEY.md §7 hard part 1):
//     pre-lock write set -> take ticket -> validate read set -> finalize ->
//     write back + release in ONE 128-bit store {value, version = ticket+1}
// The ticket is taken AFTER the write claims are visible and BEFORE the read
// set is validated, so ascending ticket order is a valid serial order: it is
// what hetm_dev_execute_batch reports and what the oracle replays.
//
// Reads take a 128-bit snapshot {value, lock}: with no FINAL bit the value is
// the one committed under that version (values only change under FINAL, and
// the release store changes value and version atomically).
// Ordering relies on value/control dependencies (a warp issues in order and
// the GPU does not speculate loads): claims are checked before the ticket is
// taken, and the ticket is broadcast with a shuffle before validation loads.
#pragma once
#include "common.cuh"

namespace hetm_b200 {

constexpr unsigned long long kLockFinal = 1ull << 63;

constexpr uint32_t kTsVersion = 0xffffffffu;  // version a TS word reads as

__device__ __forceinline__ uint32_t lk_owner(unsigned long long l) {
    return (l & kTsTag) ? 0u : (uint32_t)(l >> 32) & 0x3fffffffu;
}
__device__ __forceinline__ uint32_t lk_ver(unsigned long long l) { return (l & kTsTag) ? kTsVersion : (uint32_t)l; }
__device__ __forceinline__ unsigned long long lk_make(uint32_t owner, uint32_t ver) {
    return ((unsigned long long)owner << 32) | ver;
}
// unlocked word published by the commit holding ticket t
__device__ __forceinline__ unsigned long long lk_commit(unsigned long long t) {
    return lk_make(0, (uint32_t)((t + 1) & 0x7fffffffull));
}

template <int R, int W>
struct DeviceTx {
    uint32_t prio;
    int nr, nw;
    uint64_t r_local[R];
    uint64_t r_val[R];
    uint32_t r_ver[R];
    uint64_t w_local[W];
    uint64_t w_val[W];

    __device__ __forceinline__ void begin(uint32_t p) {
        prio = p;
        nr = 0;
        nw = 0;
    }
};

// TM_read with read-your-writes (own buffered write, then own read set).
template <int R, int W>
__device__ __forceinline__ bool tm_read(DeviceTx<R, W>& tx, const ShardView& v, uint64_t loc, uint64_t& out) {
    for (int j = 0; j < tx.nw; ++j)
        if (tx.w_local[j] == loc) { out = tx.w_val[j]; return true; }
    for (int j = 0; j < tx.nr; ++j)
        if (tx.r_local[j] == loc) { out = tx.r_val[j]; return true; }
    uint64_t val;
    unsigned long long lock;
    ld_pair(&v.cells[loc], val, lock);
    if (lock & kLockFinal) return false;
    tx.r_local[tx.nr] = loc;
    tx.r_val[tx.nr] = val;
    tx.r_ver[tx.nr] = lk_ver(lock);
    ++tx.nr;
    out = val;
    return true;
}

// TM_write: buffered; the word joins the read set first (no blind writes,
// SPEC.md:108,144).
template <int R, int W>
__device__ __forceinline__ bool tm_write(DeviceTx<R, W>& tx, const ShardView& v, uint64_t loc, uint64_t val) {
    bool in_rs = false;
    for (int j = 0; j < tx.nr; ++j) in_rs |= (tx.r_local[j] == loc);
    if (!in_rs) {
        uint64_t dummy;
        if (!tm_read(tx, v, loc, dummy)) return false;
    }
    for (int j = 0; j < tx.nw; ++j)
        if (tx.w_local[j] == loc) { tx.w_val[j] = val; return true; }
    tx.w_local[tx.nw] = loc;
    tx.w_val[tx.nw] = val;
    ++tx.nw;
    return true;
}

// Warp-aggregated ticket: one atomicAdd per converged group of lanes.  All
// participating lanes hold their pre-locks at this point, so survivors of the
// group are pairwise conflict-free and lane order is a valid tie-break.
__device__ __forceinline__ unsigned long long take_ticket(unsigned long long* ctr) {
    unsigned m = __activemask();
    unsigned leader = __ffs(m) - 1;
    unsigned long long base = 0;
    if (lane_id() == leader) base = atomicAdd(ctr, (unsigned long long)__popc(m));
    base = __shfl_sync(m, base, leader);
    unsigned below = m & ((1u << lane_id()) - 1u);
    return base + __popc(below);
}

template <int R, int W>
__device__ __forceinline__ uint32_t read_version(const DeviceTx<R, W>& tx, uint64_t loc) {
    for (int k = 0; k < tx.nr; ++k)
        if (tx.r_local[k] == loc) return tx.r_ver[k];
    return 0;
}

template <int R, int W>
__device__ __forceinline__ bool tm_commit(DeviceTx<R, W>& tx, const ShardView& v, unsigned long long* ticket_ctr,
                                          unsigned long long& ticket) {
    const uint32_t me = tx.prio;
    // 1. write set, ascending word order (tm_write deduplicates)
    uint64_t wl[W];
    uint64_t wv[W];
    uint32_t wver[W];
    const int nwl = tx.nw;
    for (int j = 0; j < nwl; ++j) {
        int p = j;
        while (p > 0 && wl[p - 1] > tx.w_local[j]) {
            wl[p] = wl[p - 1];
            wv[p] = wv[p - 1];
            wver[p] = wver[p - 1];
            --p;
        }
        wl[p] = tx.w_local[j];
        wv[p] = tx.w_val[j];
        wver[p] = read_version(tx, tx.w_local[j]);
    }
    // 2. pre-lock under the priority rule
    int held = 0;
    bool ok = true;
    for (int k = 0; k < nwl && ok; ++k) {
        unsigned long long* lw = &v.cells[wl[k]].meta;
        unsigned long long cur = ld_relaxed(lw);
        for (;;) {
            if ((cur & kLockFinal) || lk_ver(cur) != wver[k]) { ok = false; break; }
            const uint32_t own = lk_owner(cur);
            if (own != 0 && own < me) { ok = false; break; }
            const unsigned long long prev = atomicCAS(lw, cur, lk_make(me, wver[k]));
            if (prev == cur) { ++held; break; }
            cur = prev;
        }
    }
    if (!ok) {
        for (int k = 0; k < held; ++k) atomicCAS(&v.cells[wl[k]].meta, lk_make(me, wver[k]), lk_make(0, wver[k]));
        return false;
    }
    // 3. commit ticket
    const unsigned long long t = take_ticket(ticket_ctr);
    ticket = t;  // reported even if validation aborts below (write-set log slots)
    // 4. validate the read-only part of the read set (steal lower-priority pre-locks)
    uint64_t st_loc[R];
    uint32_t st_ver[R];
    int ns = 0;
    for (int k = 0; k < tx.nr && ok; ++k) {
        bool written = false;
        for (int q = 0; q < nwl; ++q) written |= (wl[q] == tx.r_local[k]);
        if (written) continue;
        unsigned long long* lw = &v.cells[tx.r_local[k]].meta;
        unsigned long long cur = ld_relaxed(lw);
        for (;;) {
            if (lk_ver(cur) != tx.r_ver[k]) { ok = false; break; }
            const uint32_t own = lk_owner(cur);
            if (own != 0 && own < me) { ok = false; break; }
            if (cur & kLockFinal) {  // lower-priority holder mid-commit: wait (waits only go down in priority)
                cur = ld_relaxed(lw);
                continue;
            }
            if (own == 0 || own == me) break;
            const unsigned long long prev = atomicCAS(lw, cur, lk_make(me, tx.r_ver[k]));
            if (prev == cur) {
                st_loc[ns] = tx.r_local[k];
                st_ver[ns] = tx.r_ver[k];
                ++ns;
                break;
            }
            cur = prev;
        }
    }
    // 5. finalize the write locks
    int fin = 0;
    if (ok) {
        for (; fin < nwl; ++fin) {
            const unsigned long long exp = lk_make(me, wver[fin]);
            if (atomicCAS(&v.cells[wl[fin]].meta, exp, exp | kLockFinal) != exp) { ok = false; break; }
        }
    }
    if (!ok) {
        for (int k = 0; k < nwl; ++k) {
            unsigned long long* lw = &v.cells[wl[k]].meta;
            if (k < fin) st_relaxed(lw, lk_make(0, wver[k]));  // held FINAL, nothing written
            else atomicCAS(lw, lk_make(me, wver[k]), lk_make(0, wver[k]));
        }
        for (int s = 0; s < ns; ++s) atomicCAS(&v.cells[st_loc[s]].meta, lk_make(me, st_ver[s]), lk_make(0, st_ver[s]));
        return false;
    }
    // 6. write back + release: one 128-bit store per written word
    for (int k = 0; k < nwl; ++k) st_pair(&v.cells[wl[k]], wv[k], lk_commit(t));
    for (int s = 0; s < ns; ++s) atomicCAS(&v.cells[st_loc[s]].meta, lk_make(me, st_ver[s]), lk_make(0, st_ver[s]));
    ticket = t;
    return true;
}

// Bitmap instrumentation of a committed transaction: reads set
// RS; writes set WS and RS; written chunks set the ChunkMap.
template <int R, int W>
__device__ __forceinline__ void tm_mark_bitmaps(const DeviceTx<R, W>& tx, const ShardView& v) {
    for (int k = 0; k < tx.nr; ++k) set_bit(v.rs, tx.r_local[k] >> v.gran_shift);
    for (int j = 0; j < tx.nw; ++j) {
        set_bit(v.ws, tx.w_local[j] >> v.gran_shift);
        set_bit(v.chunk, tx.w_local[j] >> v.chunk_shift);
    }
}

}  // namespace hetm_b200
