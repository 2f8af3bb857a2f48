// validate.cu — inter-device validation and TS-guarded apply (engine module).
//
// validateChunk: for each host write-log
// entry <addr,value,ts>:
//   (a) if the GPU read-set bit covering addr is set -> round conflictFlag;
//   (b) apply mode, regardless of (a): devReplica[addr] takes the value of the
//       freshest entry (entry.ts > TS[addr].ts).  Validate-only skips (b).
//
// Two lock-free passes per chunk replace the paper's per-entry TS lock bit
// (the lock bit of SPEC.md:320 is never needed):
//   pass A  REDG.E.MAX.64 on the word cell's `ts` (fire-and-forget),
//   pass B  the entry whose ts equals the cell's ts — the unique maximum —
//           stores its value into the same 32-B sector.
// The result equals SPEC.md:348 in any delivery order.  Apply-mode chunks are
// serialised on one stream, so every pass B sees all earlier pass A's.  The TS
// field is never reset between rounds (GlobalClock is monotone,
// SPEC.md:101-103); a ts at or below the previous rounds' maximum (ts_floor)
// is flagged instead.
#include "common.cuh"
#include "kernels.h"

#include <cstdlib>


namespace hetm_b200 {

constexpr int kValThreads = 256;
constexpr int kUnroll = 4;  // entries in flight per thread

struct EntryRegs {
    uint64_t addr, value, ts;
};

__device__ __forceinline__ EntryRegs load_entry(const hetm_log_entry* log, uint64_t i) {
    const uint64_t* e = reinterpret_cast<const uint64_t*>(log + i);
    return EntryRegs{__ldg(e), __ldg(e + 1), __ldg(e + 2)};
}

// The entries a validation launch covers: a flat array of n entries, or the
// received regions of a peer arena (region r = base[r*cap .. r*cap + counts[r]),
// counts read on the device, so the launch needs no host round trip).
// Logical index g runs over [0, total) across the regions in order.
struct LogView {
    const hetm_log_entry* base;
    uint64_t n;                             // flat entry count (segments == nullptr)
    const unsigned long long* segments;     // device counts of the regions, or nullptr
    uint32_t n_seg;                         // <= 64
    uint64_t cap;                           // entries per region
};

struct SegPrefix {  // per-block copy of the region prefix sums
    unsigned long long pre[65];
};

__device__ __forceinline__ uint64_t view_total(const LogView& lv, SegPrefix& sp) {
    if (!lv.segments) return lv.n;
    if (threadIdx.x == 0) {
        unsigned long long run = 0;
        for (uint32_t r = 0; r < lv.n_seg; ++r) {
            sp.pre[r] = run;
            const unsigned long long c = ld_relaxed(&lv.segments[r]);
            run += c < lv.cap ? c : lv.cap;
        }
        sp.pre[lv.n_seg] = run;
    }
    __syncthreads();
    return sp.pre[lv.n_seg];
}

__device__ __forceinline__ EntryRegs view_entry(const LogView& lv, const SegPrefix& sp, uint64_t g) {
    if (!lv.segments) return load_entry(lv.base, g);
    uint32_t r = 0;
    while (r + 1 < lv.n_seg && sp.pre[r + 1] <= g) ++r;
    return load_entry(lv.base, (uint64_t)r * lv.cap + (g - sp.pre[r]));
}

// Pass A of one entry (RS test + TS raise); returns nothing, folds flags.
struct PassAFlags {
    unsigned conflict = 0, bad = 0, oob = 0;
    unsigned long long maxts = 0;
};

// RS test of one entry (validate-only pass; the apply pass inlines it).
__device__ __forceinline__ void pass_a(const ShardView& v, const EntryRegs& e, uint64_t ts_floor, PassAFlags& f) {
    const uint64_t loc = e.addr - v.base;
    if (loc >= v.size_words) {
        f.oob = 1;
        return;
    }
    const uint64_t bit = loc >> v.gran_shift;
    f.conflict |= (unsigned)((v.rs[bit >> 6] >> (bit & 63)) & 1ull);  // (a) RS test
    f.bad |= (e.ts <= ts_floor);
    f.maxts = e.ts > f.maxts ? e.ts : f.maxts;
}

__device__ __forceinline__ void flush_pass_a(PassAFlags f, DevCounters* ctr) {
    const unsigned conflict = __any_sync(0xffffffffu, f.conflict);
    const unsigned bad = __any_sync(0xffffffffu, f.bad);
    const unsigned oob = __any_sync(0xffffffffu, f.oob);
    unsigned long long maxts = f.maxts;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const unsigned long long x = __shfl_xor_sync(0xffffffffu, maxts, o);
        maxts = x > maxts ? x : maxts;
    }
    if (lane_id() == 0) {
        if (conflict) atomicOr(&ctr->conflict, 1u);
        if (bad) atomicOr(&ctr->nonmonotone, 1u);
        if (oob) atomicOr(&ctr->oob, 1u);
        if (maxts) atomicMax(&ctr->round_max_ts, maxts);
    }
}

__global__ void __launch_bounds__(kValThreads) validate_kernel(ShardView v, LogView lv, DevCounters* ctr) {
    __shared__ SegPrefix sp;
    const uint64_t n = view_total(lv, sp);
    const uint64_t ts_floor = ld_relaxed(&ctr->ts_floor);
    PassAFlags f;
    const uint64_t span = (uint64_t)gridDim.x * blockDim.x * kUnroll;
    for (uint64_t i0 = (uint64_t)blockIdx.x * blockDim.x * kUnroll + threadIdx.x; i0 < n; i0 += span) {
        EntryRegs e[kUnroll];
#pragma unroll
        for (int u = 0; u < kUnroll; ++u) {
            const uint64_t i = i0 + (uint64_t)u * blockDim.x;
            e[u] = i < n ? view_entry(lv, sp, i) : EntryRegs{v.base, 0, ~0ull};
        }
#pragma unroll
        for (int u = 0; u < kUnroll; ++u)
            if (i0 + (uint64_t)u * blockDim.x < n) pass_a(v, e[u], ts_floor, f);
    }
    flush_pass_a(f, ctr);
}

// Apply pass ("if entry.ts > TS.ts: dev[addr] = value; TS.ts = ts"):
// one RETURNING atomicMax on the cell's TS; an entry that raised the TS
// stores its value into the same (now L2-resident) sector right away.  Two
// entries of one launch for the same word can race on that store; the larger
// ts then saw a TS raised THIS round (old > ts_floor) and is queued for
// restore_kernel, which re-stores it after this launch's stores completed.
// An entry whose atomic saw a stale TS (old <= ts_floor) was first in the
// atomic order, so every later entry for that word either loses (smaller ts)
// or is queued itself.  Cost per entry: one random line RMW + one L2-hit
// store; duplicates (rare under uniform access) cost one more L2 load+store.
//
// Address window [win_lo, win_hi) (local words): only entries inside it are
// processed, so a shard too large for the TLB reach (128 GiB
// of cells) is applied in a few passes over the log, each confined to a
// window of cells; out-of-shard entries are flagged by the pass with win_lo = 0.
template <int U>
__global__ void __launch_bounds__(kValThreads) apply_kernel(ShardView v, LogView lv, DevCounters* ctr,
                                                            RestoreQueue restore, uint64_t win_lo,
                                                            uint64_t win_hi) {
    __shared__ SegPrefix sp;
    const uint64_t n = view_total(lv, sp);
    const uint64_t ts_floor = ld_relaxed(&ctr->ts_floor);
    PassAFlags f;
    const uint64_t span = (uint64_t)gridDim.x * blockDim.x * U;
    for (uint64_t i0 = (uint64_t)blockIdx.x * blockDim.x * U + threadIdx.x; i0 < n; i0 += span) {
        EntryRegs e[U];
        unsigned long long old[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const uint64_t i = i0 + (uint64_t)u * blockDim.x;
            e[u] = i < n ? view_entry(lv, sp, i) : EntryRegs{v.base + v.size_words, 0, 0};
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const uint64_t loc = e[u].addr - v.base;
            old[u] = ~0ull;
            if (i0 + (uint64_t)u * blockDim.x >= n) continue;
            if (loc >= v.size_words) {
                f.oob |= win_lo == 0;
                continue;
            }
            if (loc < win_lo || loc >= win_hi) continue;  // another window's pass
            const uint64_t bit = loc >> v.gran_shift;
            f.conflict |= (unsigned)((v.rs[bit >> 6] >> (bit & 63)) & 1ull);  // (a) RS test
            f.bad |= (e[u].ts <= ts_floor);
            f.maxts = e[u].ts > f.maxts ? e[u].ts : f.maxts;
            old[u] = atomicMax(&v.cells[loc].meta, ts_meta(e[u].ts));  // (b) TS raise (a lock word < any TS word)
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            if (old[u] >= ts_meta(e[u].ts)) continue;  // lost, out of shard, or past the end
            v.cells[e[u].addr - v.base].value = e[u].value;
            if ((old[u] & kTsTag) && (old[u] & ~kTsTag) > ts_floor) {  // raced with an entry of this round
                const unsigned long long k = atomicAdd(&ctr->restore_n, 1ull);
                if (k < restore.cap) restore.idx[k] = i0 + (uint64_t)u * blockDim.x;
            }
        }
    }
    flush_pass_a(f, ctr);
}

// Exchange form of the apply pass (the product default): the whole cell
// {value, meta} is swapped with {entry.value, TS(entry.ts)} by ONE returning
// 128-bit atomic exchange (ATOMG.E.EXCH.128).  If the displaced cell H was
// fresher — meta compares higher: a TS word of a larger ts (any TS word
// outranks a batch version word, as for atomicMax), or, for equal metas, the
// larger value — the thread puts H back with a 128-bit compare-and-swap
// (ATOMG.E.CAS.128) that only replaces an older cell, retrying on the value
// it finds until H is back or the cell holds something at least as fresh.
// Invariant: the freshest (meta, value) seen so far is always in the cell or
// in a hand that will put it back, so per word the cell ends with the
// maximum over the log of (ts, value) — SPEC.md:348's freshest entry (equal ts
// on one word needs one transaction writing the word twice, which a host
// write set never holds; the tie goes to the larger value in any order).
// Cost per entry under uniform access: one random line RMW and no dependent
// second access, so no restore pass either (the atomicMax form above needs a
// dependent value store and a restore queue for same-launch races).
__device__ __forceinline__ void exch_cell(Cell* c, uint64_t v, unsigned long long m, uint64_t& ov,
                                          unsigned long long& om) {
    asm volatile("{\n\t.reg .b128 d, s;\n\tmov.b128 s, {%2, %3};\n\t"
                 "atom.relaxed.gpu.global.exch.b128 d, [%4], s;\n\tmov.b128 {%0, %1}, d;\n\t}"
                 : "=l"(ov), "=l"(om)
                 : "l"(v), "l"(m), "l"(c)
                 : "memory");
}
// 128-bit compare-and-swap of a cell; returns the cell as it was.
__device__ __forceinline__ void cas_cell(Cell* c, uint64_t ev, unsigned long long em, uint64_t v, unsigned long long m,
                                         uint64_t& ov, unsigned long long& om) {
    asm volatile("{\n\t.reg .b128 d, e, s;\n\tmov.b128 e, {%2, %3};\n\tmov.b128 s, {%4, %5};\n\t"
                 "atom.relaxed.gpu.global.cas.b128 d, [%6], e, s;\n\tmov.b128 {%0, %1}, d;\n\t}"
                 : "=l"(ov), "=l"(om)
                 : "l"(ev), "l"(em), "l"(v), "l"(m), "l"(c)
                 : "memory");
}
__device__ __forceinline__ bool fresher(unsigned long long am, uint64_t av, unsigned long long bm, uint64_t bv) {
    return am > bm || (am == bm && av > bv);
}
// Two forms, chosen per launch by the handle (RestoreQueue::amax): a log whose
// words repeat a lot (zipf host logs, BASELINE configs[2]) makes the exchange
// form ping-pong on its hot words — 128-bit atomics on one address serialise
// (cfg3 round 2.1 vs 1.0 ms) — while atomicMax lets every stale duplicate
// lose in one cheap op.  The kernel counts its put-backs (DevCounters::
// apply_dups, monotone); when the handle reads the counters and more than
// 1/64 of the entries applied since the last read needed one, the next
// launches run the atomicMax form + restore pass (capi.cu read_counters).
// Both forms leave identical cells.
template <int U>
__global__ void __launch_bounds__(kValThreads) apply_xchg_kernel(ShardView v, LogView lv, DevCounters* ctr,
                                                                 uint64_t win_lo, uint64_t win_hi) {
    __shared__ SegPrefix sp;
    const uint64_t n = view_total(lv, sp);
    const uint64_t ts_floor = ld_relaxed(&ctr->ts_floor);
    PassAFlags f;
    unsigned long long putbacks = 0;
    const uint64_t span = (uint64_t)gridDim.x * blockDim.x * U;
    for (uint64_t i0 = (uint64_t)blockIdx.x * blockDim.x * U + threadIdx.x; i0 < n; i0 += span) {
        EntryRegs e[U];
        uint64_t ov[U];
        unsigned long long om[U];
        bool live[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const uint64_t i = i0 + (uint64_t)u * blockDim.x;
            e[u] = i < n ? view_entry(lv, sp, i) : EntryRegs{v.base + v.size_words, 0, 0};
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const uint64_t loc = e[u].addr - v.base;
            live[u] = false;
            if (i0 + (uint64_t)u * blockDim.x >= n) continue;
            if (loc >= v.size_words) {
                f.oob |= win_lo == 0;
                continue;
            }
            if (loc < win_lo || loc >= win_hi) continue;  // another window's pass
            const uint64_t bit = loc >> v.gran_shift;
            f.conflict |= (unsigned)((v.rs[bit >> 6] >> (bit & 63)) & 1ull);  // (a) RS test
            f.bad |= (e[u].ts <= ts_floor);
            f.maxts = e[u].ts > f.maxts ? e[u].ts : f.maxts;
            exch_cell(&v.cells[loc], e[u].value, ts_meta(e[u].ts), ov[u], om[u]);  // (b) swap in
            live[u] = true;
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            if (!live[u]) continue;
            Cell* c = &v.cells[e[u].addr - v.base];
            // displaced a fresher cell H: put it back with a compare-and-swap
            // that only ever replaces something older than H (our own entry, or
            // whatever displaced it since)
            uint64_t cv = e[u].value;  // what we believe the cell holds
            unsigned long long cm = ts_meta(e[u].ts);
            if (!fresher(om[u], ov[u], cm, cv)) continue;
            ++putbacks;
            const uint64_t hv = ov[u];
            const unsigned long long hm = om[u];
            for (;;) {
                uint64_t pv;
                unsigned long long pm;
                cas_cell(c, cv, cm, hv, hm, pv, pm);
                if (pv == cv && pm == cm) break;      // H is back
                if (!fresher(hm, hv, pm, pv)) break;  // the cell already holds something at least as fresh
                cv = pv;
                cm = pm;
            }
        }
    }
    flush_pass_a(f, ctr);
    putbacks = warp_sum(putbacks);
    if (lane_id() == 0 && putbacks) atomicAdd(&ctr->apply_dups, putbacks);
}

// ---- TMA-staged apply (flat, 16-B aligned logs): one persistent CTA per SM
// walks tiles of kTile log entries; the tile after next is fetched into
// shared memory by the bulk-copy engine (cp.async.bulk + mbarrier, SASS
// UBLKCP) while the threads run the random TS RMWs of the current tile, so
// the streaming log read never sits in front of the atomics.  Same per-entry
// logic (and restore queue) as apply_kernel.
constexpr int kTile = 1024;                                   // entries per stage (24 KiB)
constexpr unsigned kTileBytes = kTile * sizeof(hetm_log_entry);
static_assert(kTileBytes % 16 == 0, "bulk copies move multiples of 16 B");

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.release.cta.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
    uint32_t done = 0;
    while (!done) {
        asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                     : "=r"(done)
                     : "r"(smem_u32(bar)), "r"(phase)
                     : "memory");
    }
}

__global__ void __launch_bounds__(kValThreads) apply_tma_kernel(ShardView v, const hetm_log_entry* __restrict__ log,
                                                                uint64_t n, DevCounters* ctr,
                                                                RestoreQueue restore) {
    extern __shared__ __align__(128) unsigned char apply_smem[];
    auto buf = reinterpret_cast<hetm_log_entry(*)[kTile]>(apply_smem);  // two stages
    __shared__ alignas(8) uint64_t bar[2];
    const uint64_t ts_floor = ld_relaxed(&ctr->ts_floor);
    const uint64_t full_tiles = n / kTile;  // the partial tail tile is read straight from global memory
    const uint64_t tiles = (n + kTile - 1) / kTile;
    if (threadIdx.x == 0) {
        mbar_init(&bar[0], 1);
        mbar_init(&bar[1], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    // prologue: this CTA's first two full tiles
    for (int st = 0; st < 2; ++st) {
        const uint64_t t = blockIdx.x + (uint64_t)st * gridDim.x;
        if (threadIdx.x == 0 && t < full_tiles) {
            mbar_expect_tx(&bar[st], kTileBytes);
            bulk_g2s(buf[st], log + t * kTile, kTileBytes, &bar[st]);
        }
    }
    PassAFlags f;
    uint32_t phase[2] = {0, 0};
    uint32_t it = 0;
    for (uint64_t t = blockIdx.x; t < tiles; t += gridDim.x, ++it) {
        const int st = it & 1;
        const bool staged = t < full_tiles;
        if (staged) {
            mbar_wait(&bar[st], phase[st]);
            phase[st] ^= 1;
        }
        constexpr int U = kTile / kValThreads;
        EntryRegs e[U];
        unsigned long long old[U];
        const uint64_t base_i = t * kTile;
        const uint64_t m = staged ? kTile : n - base_i;
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const uint32_t j = threadIdx.x + u * kValThreads;
            if (j < m) {
                if (staged) {
                    const hetm_log_entry& x = buf[st][j];
                    e[u] = EntryRegs{x.addr, x.value, x.ts};
                } else {
                    e[u] = load_entry(log, base_i + j);
                }
            } else {
                e[u] = EntryRegs{v.base + v.size_words, 0, 0};
            }
        }
        __syncthreads();  // every thread has its entries: the stage can be refilled
        if (threadIdx.x == 0) {
            const uint64_t nt = t + 2 * (uint64_t)gridDim.x;
            if (nt < full_tiles) {
                mbar_expect_tx(&bar[st], kTileBytes);
                bulk_g2s(buf[st], log + nt * kTile, kTileBytes, &bar[st]);
            }
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const uint64_t loc = e[u].addr - v.base;
            old[u] = ~0ull;
            if (threadIdx.x + u * kValThreads >= m) continue;
            if (loc >= v.size_words) {
                f.oob = 1;
                continue;
            }
            const uint64_t bit = loc >> v.gran_shift;
            f.conflict |= (unsigned)((v.rs[bit >> 6] >> (bit & 63)) & 1ull);  // (a) RS test
            f.bad |= (e[u].ts <= ts_floor);
            f.maxts = e[u].ts > f.maxts ? e[u].ts : f.maxts;
            old[u] = atomicMax(&v.cells[loc].meta, ts_meta(e[u].ts));  // (b) TS raise
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            if (old[u] >= ts_meta(e[u].ts)) continue;
            v.cells[e[u].addr - v.base].value = e[u].value;
            if ((old[u] & kTsTag) && (old[u] & ~kTsTag) > ts_floor) {
                const unsigned long long k = atomicAdd(&ctr->restore_n, 1ull);
                if (k < restore.cap) restore.idx[k] = base_i + threadIdx.x + u * kValThreads;
            }
        }
    }
    flush_pass_a(f, ctr);
}

// Re-store the queued entries whose ts is still the cell's TS (the unique
// freshest one per word).  If the queue overflowed, every entry of the launch
// is checked (pass B of the classic two-pass scheme).  The last block to
// finish resets the queue for the next apply launch on this stream.
__global__ void __launch_bounds__(kValThreads) restore_kernel(ShardView v, LogView lv, DevCounters* ctr,
                                                              RestoreQueue restore) {
    __shared__ SegPrefix sp;
    const uint64_t n = view_total(lv, sp);
    const unsigned long long m = ld_relaxed(&ctr->restore_n);
    const bool full = m > restore.cap;
    const uint64_t cnt = full ? n : m;
    for (uint64_t j = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; j < cnt; j += (uint64_t)gridDim.x * blockDim.x) {
        const EntryRegs e = view_entry(lv, sp, full ? j : restore.idx[j]);
        const uint64_t loc = e.addr - v.base;
        if (loc < v.size_words && ld_relaxed(&v.cells[loc].meta) == ts_meta(e.ts)) v.cells[loc].value = e.value;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        if (atomicAdd(&ctr->restore_done, 1ull) == gridDim.x - 1) {
            ctr->restore_n = 0;
            ctr->restore_done = 0;
        }
    }
}

// Pass B (dst == nullptr: into the cells' value field) and its variants for
// the shadow patch / rollback (dst = plain word array): the entry whose ts
// equals the cell's TS is the freshest one for that word.  Over a flat log or
// the received regions of a peer arena (LogView); gate != nullptr: nothing is
// done when the round has a conflict (merge staged before the host knows).
__global__ void __launch_bounds__(kValThreads) winner_kernel(Cell* cells, uint64_t* dst, uint64_t base,
                                                             uint64_t size_words, LogView lv,
                                                             const DevCounters* gate) {
    __shared__ SegPrefix sp;
    const uint64_t n = view_total(lv, sp);
    if (gate && ld_relaxed((const unsigned long long*)&gate->conflict) & 0xffffffffull) return;
    const uint64_t span = (uint64_t)gridDim.x * blockDim.x * kUnroll;
    for (uint64_t i0 = (uint64_t)blockIdx.x * blockDim.x * kUnroll + threadIdx.x; i0 < n; i0 += span) {
        EntryRegs e[kUnroll];
        unsigned long long cur[kUnroll];
#pragma unroll
        for (int u = 0; u < kUnroll; ++u) {
            const uint64_t i = i0 + (uint64_t)u * blockDim.x;
            e[u] = i < n ? view_entry(lv, sp, i) : EntryRegs{base + size_words, 0, 0};
        }
#pragma unroll
        for (int u = 0; u < kUnroll; ++u) {
            const uint64_t loc = e[u].addr - base;
            cur[u] = loc < size_words ? ld_relaxed(&cells[loc].meta) : ~0ull;
        }
#pragma unroll
        for (int u = 0; u < kUnroll; ++u) {
            if (cur[u] != ts_meta(e[u].ts)) continue;
            const uint64_t loc = e[u].addr - base;
            if (dst) dst[loc] = e[u].value;
            else cells[loc].value = e[u].value;
        }
    }
}

__global__ void popcount_kernel(const unsigned long long* __restrict__ w, uint64_t n, unsigned long long* out) {
    unsigned long long c = 0;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
        c += __popcll(w[i]);
    c = warp_sum(c);
    if (lane_id() == 0 && c) atomicAdd(out, c);
}

__global__ void or_words_kernel(unsigned long long* dst, const unsigned long long* __restrict__ src, uint64_t n) {
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
        if (src[i]) atomicOr(&dst[i], src[i]);
}

// Bitwise-OR reduction of bitmaps over NVLink (NCCL has no
// bitwise OR): words [lo, hi) of dst |= the same words of every peer bitmap,
// read through peer pointers (CUDA IPC / same-process handles of other GPUs).
// Coalesced peer loads, one plain store per word; up to 16 peers per launch.
struct PeerWords {
    const unsigned long long* p[16];
};
__global__ void or_peers_kernel(unsigned long long* dst, PeerWords peers, uint32_t n_peers, uint64_t lo, uint64_t hi) {
    for (uint64_t i = lo + (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < hi; i += (uint64_t)gridDim.x * blockDim.x) {
        unsigned long long acc = dst[i];
        for (uint32_t k = 0; k < n_peers; ++k) acc |= peers.p[k][i];
        dst[i] = acc;
    }
}

static unsigned grid_cap(uint64_t items, int threads, const LaunchGeom& g, int per_sm) {
    uint64_t want = (items + threads - 1) / threads;
    const uint64_t cap = (uint64_t)per_sm * (uint64_t)g.sm_count;
    if (want > cap) want = cap;
    return (unsigned)(want ? want : 1);
}

// Rollback helpers (optimized mergeAbortDevice) and the literal
// TS reset.  0x00000000ffffffff is the unlocked reserved-version
// word a TS word reads as (device_tm.cuh), so the batch TM sees no change.
constexpr unsigned long long kUntagged = 0xffffffffull;

__global__ void untag_log_kernel(Cell* cells, uint64_t base, uint64_t size_words, LogView lv) {
    __shared__ SegPrefix sp;
    const uint64_t n = view_total(lv, sp);
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t loc = view_entry(lv, sp, i).addr - base;
        if (loc < size_words) cells[loc].meta = kUntagged;
    }
}

__global__ void log_to_shadow_kernel(uint64_t* shadow, const Cell* __restrict__ cells, uint64_t base,
                                     uint64_t size_words, LogView lv) {
    __shared__ SegPrefix sp;
    const uint64_t n = view_total(lv, sp);
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t loc = view_entry(lv, sp, i).addr - base;
        if (loc < size_words) shadow[loc] = cells[loc].value;
    }
}

__global__ void reset_ts_kernel(Cell* cells, uint64_t size_words) {
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < size_words;
         i += (uint64_t)gridDim.x * blockDim.x)
        if (cells[i].meta & kTsTag) cells[i].meta = kUntagged;
}

cudaError_t launch_reset_ts(Cell* cells, uint64_t size_words, const LaunchGeom& g, cudaStream_t s) {
    reset_ts_kernel<<<(unsigned)g.sm_count * 8u, kValThreads, 0, s>>>(cells, size_words);
    return cudaGetLastError();
}

// Round boundary on the device: ts_floor = max(ts_floor, round_max_ts) (or 0
// for the literal SPEC.md:421 TS reset), round_max_ts = 0.  Enqueued by both
// the synchronous and the asynchronous clear so pipelined rounds keep an exact
// floor without a host round trip.
// clearRound in one launch, stream-ordered behind the round's
// work: zero RS, WS and ChunkMap, clear the round's conflict / nonmonotone /
// out-of-shard flags and roll the round counters (block 0): TS floor = max ts
// seen so far, the next round's write-set log starts at the current ticket.
__global__ void clear_round_kernel(unsigned long long* rs, unsigned long long* ws, uint64_t rs_words,
                                   unsigned long long* chunk, uint64_t chunk_words, DevCounters* ctr, int reset_ts) {
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        const unsigned long long m = ctr->round_max_ts;
        ctr->ts_floor = reset_ts ? 0ull : (m > ctr->ts_floor ? m : ctr->ts_floor);
        ctr->round_max_ts = 0;
        ctr->wlog_base = ctr->ticket;
        ctr->wlog_overflow = 0;
        ctr->conflict = 0;
        ctr->nonmonotone = 0;
        ctr->oob = 0;
    }
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < rs_words; i += stride) {
        rs[i] = 0;
        ws[i] = 0;
    }
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < chunk_words; i += stride) chunk[i] = 0;
}

cudaError_t launch_clear_round(unsigned long long* rs, unsigned long long* ws, uint64_t rs_words,
                               unsigned long long* chunk, uint64_t chunk_words, DevCounters* ctr, int reset_ts,
                               const LaunchGeom& g, cudaStream_t s) {
    const uint64_t n = rs_words > chunk_words ? rs_words : chunk_words;
    clear_round_kernel<<<grid_cap(n ? n : 1, 256, g, 2), 256, 0, s>>>(rs, ws, rs_words, chunk, chunk_words, ctr,
                                                                      reset_ts);
    return cudaGetLastError();
}

// Core launcher over a LogView; n_hint sizes the grid (the flat count, or the
// segmented view's capacity when the counts live on the device).
static cudaError_t launch_view(const ShardView& v, const LogView& lv, uint64_t n_hint, int apply, DevCounters* ctr,
                               RestoreQueue rq, const LaunchGeom& g, cudaStream_t s) {
    if (n_hint == 0) return cudaSuccess;
    const unsigned grid = grid_cap((n_hint + kUnroll - 1) / kUnroll, kValThreads, g, g.max_blocks_val);
    if (!apply) {
        validate_kernel<<<grid, kValThreads, 0, s>>>(v, lv, ctr);
        return cudaGetLastError();
    }
    static const int apply_bps = [] {  // tuning experiments only: resident blocks per SM for apply
        const char* e = std::getenv("HETM_APPLY_BLOCKS_PER_SM");
        return e ? std::atoi(e) : 0;
    }();
    static const int apply_unroll = [] {  // tuning experiments only: entries in flight per thread
        const char* e = std::getenv("HETM_APPLY_UNROLL");
        return e ? std::atoi(e) : 4;
    }();
    // one resident CTA per SM: fewer random RMWs in flight queue less (measured
    // 0.081 vs 0.111 ms per 2^20 entries at full occupancy)
    const int bps = apply_bps > 0 ? apply_bps : 1;
    const int u = apply_unroll == 2 || apply_unroll == 8 ? apply_unroll : 4;
    const unsigned agrid = grid_cap((n_hint + u - 1) / u, kValThreads, g, bps);
    static const bool tma = [] {  // experiment only (HETM_APPLY_TMA=1): measured no faster, profiles/r01_apply_tma.txt
        const char* e = std::getenv("HETM_APPLY_TMA");
        return e && std::atoi(e) != 0;
    }();
    if (tma && !lv.segments && (reinterpret_cast<uintptr_t>(lv.base) & 15) == 0 && n_hint >= (uint64_t)kTile) {
        const uint64_t tiles = (n_hint + kTile - 1) / kTile;
        const unsigned tgrid = (unsigned)(tiles < (uint64_t)g.sm_count ? tiles : (uint64_t)g.sm_count);
        static const cudaError_t attr =
            cudaFuncSetAttribute(apply_tma_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 2 * kTileBytes);
        if (attr != cudaSuccess) return attr;
        apply_tma_kernel<<<tgrid, kValThreads, 2 * kTileBytes, s>>>(v, lv.base, n_hint, ctr, rq);
        restore_kernel<<<2 * g.sm_count, kValThreads, 0, s>>>(v, lv, ctr, rq);
        return cudaGetLastError();
    }
    // Address windows: random 16-B cells over more than 64 GiB of cells outrun
    // the TLB reach (5 G entries/s on a 64 GiB shard = 128 GiB of cells vs 13
    // on 32 GiB; profiles/r02c_bucket_probe.txt), so such shards are applied
    // in passes over the log, each confined to 2^32 words (64 GiB of cells):
    // 14.5 G entries/s on the 64 GiB shard (windows of 2^31: 10.1, 2^30: 5.8;
    // profiles/r02d_window_probe.txt).
    static const uint32_t win_log2 = [] {  // tuning experiments only: HETM_APPLY_WINDOW_LOG2
        const char* e = std::getenv("HETM_APPLY_WINDOW_LOG2");
        return e ? (uint32_t)std::atoi(e) : 32u;
    }();
    static const uint64_t win_min_shard = [] {  // shards above this many words are windowed
        const char* e = std::getenv("HETM_APPLY_WINDOW_ABOVE_LOG2");
        return 1ull << (e ? std::atoi(e) : 32);
    }();
    const uint64_t win = v.size_words > win_min_shard && win_log2 < 40 ? (1ull << win_log2) : v.size_words;
    static const bool amax = [] {  // A/B only (HETM_APPLY_AMAX=1): always the atomicMax + restore form
        // (otherwise the handle picks it per launch for hot logs: RestoreQueue::amax)
        const char* e = std::getenv("HETM_APPLY_AMAX");
        return e && std::atoi(e) != 0;
    }();
    if (!amax && !rq.amax) {  // the exchange form (apply_xchg_kernel): no restore pass
        for (uint64_t lo = 0; lo < v.size_words; lo += win) {
            const uint64_t hi = v.size_words - lo > win ? lo + win : v.size_words;
            if (u == 2) apply_xchg_kernel<2><<<agrid, kValThreads, 0, s>>>(v, lv, ctr, lo, hi);
            else if (u == 8) apply_xchg_kernel<8><<<agrid, kValThreads, 0, s>>>(v, lv, ctr, lo, hi);
            else apply_xchg_kernel<4><<<agrid, kValThreads, 0, s>>>(v, lv, ctr, lo, hi);
        }
        return cudaGetLastError();
    }
    for (uint64_t lo = 0; lo < v.size_words; lo += win) {
        const uint64_t hi = v.size_words - lo > win ? lo + win : v.size_words;
        if (u == 2) apply_kernel<2><<<agrid, kValThreads, 0, s>>>(v, lv, ctr, rq, lo, hi);
        else if (u == 8) apply_kernel<8><<<agrid, kValThreads, 0, s>>>(v, lv, ctr, rq, lo, hi);
        else apply_kernel<4><<<agrid, kValThreads, 0, s>>>(v, lv, ctr, rq, lo, hi);
    }
    restore_kernel<<<2 * g.sm_count, kValThreads, 0, s>>>(v, lv, ctr, rq);
    return cudaGetLastError();
}

// Fault injection only (HETM_FAULT_SKIP_TS, the checker's mutation suite,
// SPEC.md:569): every entry is stored in arrival order, with no TS freshness
// test, so an older host write can overwrite a newer one.
__global__ void blind_apply_kernel(ShardView v, const hetm_log_entry* __restrict__ log, uint64_t n, DevCounters* ctr) {
    const uint64_t ts_floor = ld_relaxed(&ctr->ts_floor);
    PassAFlags f;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
        const EntryRegs e = load_entry(log, i);
        pass_a(v, e, ts_floor, f);
        const uint64_t loc = e.addr - v.base;
        if (loc < v.size_words) {
            v.cells[loc].value = e.value;
            v.cells[loc].meta = ts_meta(e.ts);
        }
    }
    flush_pass_a(f, ctr);
}

cudaError_t launch_blind_apply(const ShardView& v, const hetm_log_entry* d_log, uint64_t n, DevCounters* ctr,
                               const LaunchGeom& g, cudaStream_t s) {
    if (n == 0) return cudaSuccess;
    blind_apply_kernel<<<grid_cap(n, kValThreads, g, 4), kValThreads, 0, s>>>(v, d_log, n, ctr);
    return cudaGetLastError();
}

cudaError_t launch_validate(const ShardView& v, const hetm_log_entry* d_log, uint64_t n, int apply,
                            DevCounters* ctr, RestoreQueue rq, const LaunchGeom& g, cudaStream_t s) {
    return launch_view(v, LogView{d_log, n, nullptr, 0, 0}, n, apply, ctr, rq, g, s);
}

cudaError_t launch_validate_regions(const ShardView& v, const hetm_log_entry* d_base, const unsigned long long* d_counts,
                                    uint32_t n_regions, uint64_t cap, int apply, DevCounters* ctr,
                                    RestoreQueue rq, const LaunchGeom& g, cudaStream_t s) {
    if (n_regions == 0 || n_regions > 64) return cudaErrorInvalidValue;
    // the grid is sized for one region's worth (the expected share); the kernels grid-stride over the total
    return launch_view(v, LogView{d_base, 0, d_counts, n_regions, cap}, cap, apply, ctr, rq, g, s);
}

// Clean re-apply of the round's host log (the arena and any received peer
// regions) onto the device replica whose device write set was restored from
// devShadow: forget this round's TS words of every logged word first (a batch
// that ran after an earlier apply may have replaced some), then apply all the
// logs (apply + restore kernels), then copy the logged words to devShadow.
cudaError_t launch_rollback_reapply(const ShardView& v, uint64_t* shadow, const RoundLogs& logs, DevCounters* ctr,
                                    RestoreQueue rq, const LaunchGeom& g, cudaStream_t s) {
    for (int pass = 0; pass < 3; ++pass) {
        for (uint32_t k = 0; k <= logs.n_regions_sets; ++k) {
            const bool flat = k == 0;
            if (flat && logs.n == 0) continue;
            const LogView lv = flat ? LogView{logs.flat, logs.n, nullptr, 0, 0}
                                    : LogView{logs.region[k - 1].base, 0, logs.region[k - 1].counts,
                                              logs.region[k - 1].n_regions, logs.region[k - 1].cap};
            const uint64_t hint = flat ? logs.n : lv.cap;
            const unsigned grid = grid_cap(hint, kValThreads, g, 8);
            if (pass == 0) {
                untag_log_kernel<<<grid, kValThreads, 0, s>>>(v.cells, v.base, v.size_words, lv);
            } else if (pass == 1) {
                cudaError_t e = launch_view(v, lv, hint, 1, ctr, rq, g, s);
                if (e != cudaSuccess) return e;
            } else if (shadow) {
                log_to_shadow_kernel<<<grid, kValThreads, 0, s>>>(shadow, v.cells, v.base, v.size_words, lv);
            }
        }
    }
    return cudaGetLastError();
}

cudaError_t launch_winner_apply(Cell* cells, uint64_t* dst, uint64_t base, uint64_t size_words,
                                const hetm_log_entry* d_log, uint64_t n, const LaunchGeom& g, cudaStream_t s,
                                const DevCounters* gate) {
    if (n == 0) return cudaSuccess;
    const unsigned grid = grid_cap((n + kUnroll - 1) / kUnroll, kValThreads, g, g.max_blocks_val);
    winner_kernel<<<grid, kValThreads, 0, s>>>(cells, dst, base, size_words, LogView{d_log, n, nullptr, 0, 0}, gate);
    return cudaGetLastError();
}

cudaError_t launch_winner_regions(Cell* cells, uint64_t* dst, uint64_t base, uint64_t size_words,
                                  const hetm_log_entry* d_base, const unsigned long long* d_counts,
                                  uint32_t n_regions, uint64_t cap, const LaunchGeom& g, cudaStream_t s,
                                  const DevCounters* gate) {
    if (n_regions == 0 || n_regions > 64) return cudaErrorInvalidValue;
    const unsigned grid = grid_cap((cap + kUnroll - 1) / kUnroll, kValThreads, g, g.max_blocks_val);
    winner_kernel<<<grid, kValThreads, 0, s>>>(cells, dst, base, size_words,
                                               LogView{d_base, 0, d_counts, n_regions, cap}, gate);
    return cudaGetLastError();
}

cudaError_t launch_popcount(const unsigned long long* w, uint64_t n, unsigned long long* out, cudaStream_t s) {
    if (n == 0) return cudaSuccess;
    uint64_t grid = (n + 255) / 256;
    if (grid > 1184) grid = 1184;
    popcount_kernel<<<(unsigned)grid, 256, 0, s>>>(w, n, out);
    return cudaGetLastError();
}

cudaError_t launch_or_words(unsigned long long* dst, const unsigned long long* src, uint64_t n, cudaStream_t s) {
    if (n == 0) return cudaSuccess;
    uint64_t grid = (n + 255) / 256;
    if (grid > 1184) grid = 1184;
    or_words_kernel<<<(unsigned)grid, 256, 0, s>>>(dst, src, n);
    return cudaGetLastError();
}

cudaError_t launch_or_peers(unsigned long long* dst, const unsigned long long* const* peers, uint32_t n_peers,
                            uint64_t lo, uint64_t hi, const LaunchGeom& g, cudaStream_t s) {
    if (hi <= lo || n_peers == 0) return cudaSuccess;
    for (uint32_t base = 0; base < n_peers; base += 16) {
        PeerWords pw{};
        const uint32_t m = n_peers - base < 16 ? n_peers - base : 16;
        for (uint32_t k = 0; k < m; ++k) pw.p[k] = peers[base + k];
        or_peers_kernel<<<grid_cap(hi - lo, 256, g, 8), 256, 0, s>>>(dst, pw, m, lo, hi);
    }
    return cudaGetLastError();
}

int query_val_occupancy(int* blocks) {
    int b = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, validate_kernel, kValThreads, 0) != cudaSuccess)
        return -1;
    *blocks = b;
    return 0;
}

}  // namespace hetm_b200
