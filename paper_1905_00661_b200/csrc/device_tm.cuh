// device_tm.cuh — PR-STM-style device guest TM.
//
// Device-side TM_read / TM_write / TM_commit for transactional kernels.  One
// CUDA thread runs one transaction; every transaction eventually commits or
// reports livelock.
//
// Lock table: 64-bit versioned locks, one per (hashed) STMR word:
//     bit 63      FINAL  — write-back in progress, never stolen
//     bits 62..32 owner  — priority of the pre-lock holder (0 = free)
//     bits 31..0  version — low 32 bits of the last committing ticket + 1
// Priority rule (PR-STM): priority = batch index + 1, smaller wins.  A
// transaction may steal a lower-priority PRE-lock; the robbed transaction
// fails its finalize step and retries.  The highest-priority live transaction
// is therefore only ever aborted by a FINAL lock (its holder is already
// writing back) or by a version change (someone committed): no livelock.
//
// Commit (TL2 order, SURVEY.md §7 hard part 1):
//     pre-lock write set -> take ticket -> validate read set -> finalize ->
//     write back -> release (version = ticket + 1)
// The ticket is taken AFTER the write claims are visible and BEFORE the read
// set is validated, so ascending ticket order is a valid serial order: it is
// what hetm_dev_execute_batch reports and what the oracle replays.
//
// Ordering on sm_100a relies on value/control dependencies (the GPU issues a
// warp's instructions in order and does not speculate loads):
//   * lock words are loaded and tested before the dependent STMR loads issue;
//   * the ticket is broadcast with a shuffle before validation loads issue;
//   * write-back stores are fenced (fence.acq_rel.gpu) before the release.
#pragma once
#include "common.cuh"

namespace hetm_b200 {

constexpr unsigned long long kLockFinal = 1ull << 63;

__device__ __forceinline__ uint32_t lk_owner(unsigned long long l) { return (uint32_t)(l >> 32) & 0x7fffffffu; }
__device__ __forceinline__ uint32_t lk_ver(unsigned long long l) { return (uint32_t)l; }
__device__ __forceinline__ unsigned long long lk_make(uint32_t owner, uint32_t ver) {
    return ((unsigned long long)owner << 32) | ver;
}

struct LockTable {
    unsigned long long* words;
    uint32_t hash_shift;  // 64 - log2(entries)
    uint32_t identity;    // 1: one lock per local word (entries >= size_words)
    __device__ __forceinline__ uint32_t index(uint64_t local) const {
        return identity ? (uint32_t)local : (uint32_t)((local * 0x9E3779B97F4A7C15ull) >> hash_shift);
    }
};

template <int R, int W>
struct DeviceTx {
    uint32_t prio;
    int nr, nw;
    uint64_t r_local[R];
    uint64_t r_val[R];
    uint32_t r_lk[R];
    uint32_t r_ver[R];
    uint64_t w_local[W];
    uint64_t w_val[W];

    __device__ __forceinline__ void begin(uint32_t p) {
        prio = p;
        nr = 0;
        nw = 0;
    }
};

// Batched TM_read of n words (local indices).  Lock words of all n are loaded
// first (in parallel); the STMR loads are control-dependent on them.  Returns
// false (abort) if any is FINAL-locked.  No read-your-writes lookup: use
// tm_read for words that may already be in the write buffer.
template <int R, int W, int N>
__device__ __forceinline__ bool tm_read_n(DeviceTx<R, W>& tx, const ShardView& v, const LockTable& lt,
                                          const uint64_t (&loc)[N], uint64_t (&out)[N]) {
    unsigned long long l[N];
    uint32_t lk[N];
#pragma unroll
    for (int k = 0; k < N; ++k) {
        lk[k] = lt.index(loc[k]);
        l[k] = ld_relaxed(&lt.words[lk[k]]);
    }
    bool fin = false;
#pragma unroll
    for (int k = 0; k < N; ++k) fin |= (l[k] & kLockFinal) != 0;
    if (fin) return false;
#pragma unroll
    for (int k = 0; k < N; ++k) out[k] = ld_relaxed(&v.stmr[loc[k]]);
#pragma unroll
    for (int k = 0; k < N; ++k) {
        tx.r_local[tx.nr] = loc[k];
        tx.r_val[tx.nr] = out[k];
        tx.r_lk[tx.nr] = lk[k];
        tx.r_ver[tx.nr] = lk_ver(l[k]);
        ++tx.nr;
    }
    return true;
}

// Single TM_read with read-your-writes (own buffered write, then own read set).
template <int R, int W>
__device__ __forceinline__ bool tm_read(DeviceTx<R, W>& tx, const ShardView& v, const LockTable& lt,
                                        uint64_t loc, uint64_t& out) {
    for (int j = 0; j < tx.nw; ++j)
        if (tx.w_local[j] == loc) { out = tx.w_val[j]; return true; }
    for (int j = 0; j < tx.nr; ++j)
        if (tx.r_local[j] == loc) { out = tx.r_val[j]; return true; }
    uint64_t a[1] = {loc}, o[1];
    if (!tm_read_n(tx, v, lt, a, o)) return false;
    out = o[0];
    return true;
}

// TM_write: buffered; the word must be in the read set (no blind writes,
// SPEC.md:108,144) — callers read first, tm_write enforces it.
template <int R, int W>
__device__ __forceinline__ bool tm_write(DeviceTx<R, W>& tx, const ShardView& v, const LockTable& lt,
                                         uint64_t loc, uint64_t val) {
    bool in_rs = false;
    for (int j = 0; j < tx.nr; ++j) in_rs |= (tx.r_local[j] == loc);
    if (!in_rs) {
        uint64_t dummy;
        if (!tm_read(tx, v, lt, loc, dummy)) return false;
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
__device__ __forceinline__ bool tm_commit(DeviceTx<R, W>& tx, const ShardView& v, const LockTable& lt,
                                          unsigned long long* ticket_ctr, unsigned long long& ticket) {
    const uint32_t me = tx.prio;
    // 0. words sharing a lock entry must have been read under one version
    for (int k = 1; k < tx.nr; ++k)
        for (int q = 0; q < k; ++q)
            if (tx.r_lk[q] == tx.r_lk[k] && tx.r_ver[q] != tx.r_ver[k]) return false;
    // 1. write lock set (distinct lock indices, ascending) with read versions
    uint32_t wl[W], wv[W];
    int nwl = 0;
    for (int j = 0; j < tx.nw; ++j) {
        uint32_t lk = lt.index(tx.w_local[j]);
        uint32_t ver = 0;
        for (int k = 0; k < tx.nr; ++k)
            if (tx.r_lk[k] == lk) { ver = tx.r_ver[k]; break; }
        bool dup = false;
        for (int k = 0; k < nwl; ++k) dup |= (wl[k] == lk);
        if (dup) continue;
        int p = nwl++;
        while (p > 0 && wl[p - 1] > lk) { wl[p] = wl[p - 1]; wv[p] = wv[p - 1]; --p; }
        wl[p] = lk;
        wv[p] = ver;
    }
    // 2. pre-lock under the priority rule
    int held = 0;
    bool ok = true;
    for (int k = 0; k < nwl && ok; ++k) {
        unsigned long long want = lk_make(me, wv[k]);
        unsigned long long cur = ld_relaxed(&lt.words[wl[k]]);
        for (;;) {
            if ((cur & kLockFinal) || lk_ver(cur) != wv[k]) { ok = false; break; }
            uint32_t own = lk_owner(cur);
            if (own != 0 && own < me) { ok = false; break; }
            unsigned long long prev = atomicCAS(&lt.words[wl[k]], cur, want);
            if (prev == cur) { ++held; break; }
            cur = prev;
        }
    }
    if (!ok) {
        for (int k = 0; k < held; ++k) atomicCAS(&lt.words[wl[k]], lk_make(me, wv[k]), lk_make(0, wv[k]));
        return false;
    }
    // 3. commit ticket
    const unsigned long long t = take_ticket(ticket_ctr);
    // 4. validate the read-only part of the read set (steal lower-priority pre-locks)
    uint32_t st_lk[R], st_ver[R];
    int ns = 0;
    for (int k = 0; k < tx.nr && ok; ++k) {
        uint32_t lk = tx.r_lk[k];
        bool skip = false;
        for (int q = 0; q < nwl; ++q) skip |= (wl[q] == lk);
        for (int q = 0; q < k; ++q) skip |= (tx.r_lk[q] == lk);
        if (skip) continue;
        unsigned long long cur = ld_relaxed(&lt.words[lk]);
        for (;;) {
            if ((cur & kLockFinal) || lk_ver(cur) != tx.r_ver[k]) { ok = false; break; }
            uint32_t own = lk_owner(cur);
            if (own == 0 || own == me) break;
            if (own < me) { ok = false; break; }
            unsigned long long prev = atomicCAS(&lt.words[lk], cur, lk_make(me, tx.r_ver[k]));
            if (prev == cur) { st_lk[ns] = lk; st_ver[ns] = tx.r_ver[k]; ++ns; break; }
            cur = prev;
        }
    }
    // 5. finalize the write locks
    int fin = 0;
    if (ok) {
        for (; fin < nwl; ++fin) {
            unsigned long long exp = lk_make(me, wv[fin]);
            if (atomicCAS(&lt.words[wl[fin]], exp, exp | kLockFinal) != exp) { ok = false; break; }
        }
    }
    if (!ok) {
        for (int k = 0; k < nwl; ++k) {
            if (k < fin) st_relaxed(&lt.words[wl[k]], lk_make(0, wv[k]));  // held FINAL, nothing written
            else atomicCAS(&lt.words[wl[k]], lk_make(me, wv[k]), lk_make(0, wv[k]));
        }
        for (int s = 0; s < ns; ++s) atomicCAS(&lt.words[st_lk[s]], lk_make(me, st_ver[s]), lk_make(0, st_ver[s]));
        return false;
    }
    // 6. write back, then release with the new version
    for (int j = 0; j < tx.nw; ++j) st_relaxed(&v.stmr[tx.w_local[j]], tx.w_val[j]);
    fence_acq_rel();
    const uint32_t nv = (uint32_t)(t + 1);
    for (int k = 0; k < nwl; ++k) st_relaxed(&lt.words[wl[k]], lk_make(0, nv));
    for (int s = 0; s < ns; ++s) atomicCAS(&lt.words[st_lk[s]], lk_make(me, st_ver[s]), lk_make(0, st_ver[s]));
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
