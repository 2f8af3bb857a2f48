// validate.cu — inter-device validation and TS-guarded apply (engine module).
// (the TS lock bit of SPEC.md:320 is kept in the word layout but never set:
//  the two-pass max/winner scheme below needs no lock.)
//
// validateChunk: for each host write-log
// entry <addr,value,ts>:
//   (a) if the GPU read-set bit covering addr is set -> round conflictFlag;
//   (b) apply mode, regardless of (a): take the TS lock bit of addr; if
//       entry.ts > TS[addr].ts then devReplica[addr] = value and TS = ts;
//       release.  Validate-only mode (early validation) skips (b).
// The TS array is never reset between rounds (GlobalClock is monotone,
// SPEC.md:101-103); a ts at or below the previous rounds' maximum
// (ts_floor) is flagged instead.
#include "common.cuh"
#include "kernels.h"

namespace hetm_b200 {

constexpr int kValThreads = 256;
constexpr unsigned long long kTsLock = 1ull << 63;  // TsArray lockBit

// Two lock-free passes per chunk replace the paper's per-entry TS lock bit
// (PAPER.md:330): pass A raises TS[addr] to the freshest ts with a
// fire-and-forget REDG.E.MAX.64; pass B stores the value of the entry whose ts
// equals TS[addr] — the unique maximum, so the outcome equals SPEC.md:348's
// "apply iff entry.ts > TS.ts" in any delivery order.  Apply-mode chunks are
// serialised on one stream, so every pass B sees all earlier pass A's.
constexpr int kUnroll = 4;

struct EntryRegs {
    uint64_t addr, value, ts;
};

__device__ __forceinline__ EntryRegs load_entry(const hetm_log_entry* log, uint64_t i) {
    const uint64_t* e = reinterpret_cast<const uint64_t*>(log + i);
    return EntryRegs{__ldg(e), __ldg(e + 1), __ldg(e + 2)};
}

template <bool kApply>
__global__ void __launch_bounds__(kValThreads) validate_kernel(ShardView v, unsigned long long* ts_arr,
                                                               const hetm_log_entry* __restrict__ log, uint64_t n,
                                                               uint64_t ts_floor, DevCounters* ctr) {
    unsigned conflict = 0, bad = 0, oob = 0;
    unsigned long long maxts = 0;
    const uint64_t span = (uint64_t)gridDim.x * blockDim.x * kUnroll;
    for (uint64_t i0 = (uint64_t)blockIdx.x * blockDim.x * kUnroll + threadIdx.x; i0 < n; i0 += span) {
        EntryRegs e[kUnroll];
#pragma unroll
        for (int u = 0; u < kUnroll; ++u) {
            const uint64_t i = i0 + (uint64_t)u * blockDim.x;
            e[u] = i < n ? load_entry(log, i) : EntryRegs{v.base + v.size_words, 0, 0};
        }
#pragma unroll
        for (int u = 0; u < kUnroll; ++u) {
            if (i0 + (uint64_t)u * blockDim.x >= n) continue;
            const uint64_t loc = e[u].addr - v.base;
            if (loc >= v.size_words) { oob = 1; continue; }
            const uint64_t bit = loc >> v.gran_shift;
            conflict |= (unsigned)((v.rs[bit >> 6] >> (bit & 63)) & 1ull);  // (a) RS test
            bad |= (e[u].ts <= ts_floor);
            maxts = e[u].ts > maxts ? e[u].ts : maxts;
            if (kApply) atomicMax(&ts_arr[loc], (unsigned long long)e[u].ts);  // (b) pass A
        }
    }
    conflict = __any_sync(0xffffffffu, conflict);
    bad = __any_sync(0xffffffffu, bad);
    oob = __any_sync(0xffffffffu, oob);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        unsigned long long x = __shfl_xor_sync(0xffffffffu, maxts, o);
        maxts = x > maxts ? x : maxts;
    }
    if (lane_id() == 0) {
        if (conflict) atomicOr(&ctr->conflict, 1u);
        if (bad) atomicOr(&ctr->nonmonotone, 1u);
        if (oob) atomicOr(&ctr->oob, 1u);
        if (maxts) atomicMax(&ctr->round_max_ts, maxts);
    }
}

// Pass B / rollback / shadow patch: dst[addr] = value iff TS[addr] == ts.
__global__ void __launch_bounds__(kValThreads) winner_apply_kernel(uint64_t* dst, uint64_t base, uint64_t size_words,
                                                                   const unsigned long long* __restrict__ ts_arr,
                                                                   const hetm_log_entry* __restrict__ log, uint64_t n) {
    const uint64_t span = (uint64_t)gridDim.x * blockDim.x * kUnroll;
    for (uint64_t i0 = (uint64_t)blockIdx.x * blockDim.x * kUnroll + threadIdx.x; i0 < n; i0 += span) {
        EntryRegs e[kUnroll];
        unsigned long long cur[kUnroll];
#pragma unroll
        for (int u = 0; u < kUnroll; ++u) {
            const uint64_t i = i0 + (uint64_t)u * blockDim.x;
            e[u] = i < n ? load_entry(log, i) : EntryRegs{base + size_words, 0, 0};
        }
#pragma unroll
        for (int u = 0; u < kUnroll; ++u) {
            const uint64_t loc = e[u].addr - base;
            cur[u] = loc < size_words ? ld_relaxed(&ts_arr[loc]) : ~0ull;
        }
#pragma unroll
        for (int u = 0; u < kUnroll; ++u)
            if ((cur[u] & ~kTsLock) == e[u].ts) dst[e[u].addr - base] = e[u].value;
    }
}

// One CTA per dirty chunk at a time; 16-B vector copies.
__global__ void copy_dirty_chunks_kernel(uint64_t* __restrict__ dst, const uint64_t* __restrict__ src,
                                         uint64_t size_words, const unsigned long long* __restrict__ bits,
                                         uint64_t n_chunks, uint32_t chunk_shift) {
    const uint64_t words_per_chunk = 1ull << chunk_shift;
    for (uint64_t c = blockIdx.x; c < n_chunks; c += gridDim.x) {
        if (!((bits[c >> 6] >> (c & 63)) & 1ull)) continue;
        const uint64_t lo = c * words_per_chunk;
        uint64_t hi = lo + words_per_chunk;
        if (hi > size_words) hi = size_words;
        const uint64_t n2 = (hi - lo) / 2;
        const uint4* s4 = reinterpret_cast<const uint4*>(src + lo);
        uint4* d4 = reinterpret_cast<uint4*>(dst + lo);
        for (uint64_t k = threadIdx.x; k < n2; k += blockDim.x) d4[k] = s4[k];
        if (((hi - lo) & 1) && threadIdx.x == 0) dst[hi - 1] = src[hi - 1];
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

static unsigned grid_cap(uint64_t n, int threads, const LaunchGeom& g, int per_sm) {
    uint64_t want = (n + threads - 1) / threads;
    uint64_t cap = (uint64_t)per_sm * (uint64_t)g.sm_count;
    if (want > cap) want = cap;
    return (unsigned)(want ? want : 1);
}

cudaError_t launch_validate(const ShardView& v, unsigned long long* d_ts, const hetm_log_entry* d_log, uint64_t n,
                            int apply, uint64_t ts_floor, DevCounters* ctr, const LaunchGeom& g, cudaStream_t s) {
    if (n == 0) return cudaSuccess;
    const unsigned grid = grid_cap((n + kUnroll - 1) / kUnroll, kValThreads, g, g.max_blocks_val);
    if (apply) {
        validate_kernel<true><<<grid, kValThreads, 0, s>>>(v, d_ts, d_log, n, ts_floor, ctr);
        winner_apply_kernel<<<grid, kValThreads, 0, s>>>(v.stmr, v.base, v.size_words, d_ts, d_log, n);
    } else {
        validate_kernel<false><<<grid, kValThreads, 0, s>>>(v, d_ts, d_log, n, ts_floor, ctr);
    }
    return cudaGetLastError();
}

cudaError_t launch_winner_apply(uint64_t* dst, uint64_t base, uint64_t size_words, const unsigned long long* d_ts,
                                const hetm_log_entry* d_log, uint64_t n, const LaunchGeom& g, cudaStream_t s) {
    if (n == 0) return cudaSuccess;
    winner_apply_kernel<<<grid_cap((n + kUnroll - 1) / kUnroll, kValThreads, g, g.max_blocks_val), kValThreads, 0, s>>>(
        dst, base, size_words, d_ts, d_log, n);
    return cudaGetLastError();
}

cudaError_t launch_copy_dirty_chunks(uint64_t* dst, const uint64_t* src, uint64_t size_words,
                                     const unsigned long long* bits, uint64_t n_chunks, uint32_t chunk_shift,
                                     const LaunchGeom& g, cudaStream_t s) {
    if (n_chunks == 0) return cudaSuccess;
    uint64_t grid = n_chunks < (uint64_t)g.sm_count * 8 ? n_chunks : (uint64_t)g.sm_count * 8;
    copy_dirty_chunks_kernel<<<(unsigned)grid, 256, 0, s>>>(dst, src, size_words, bits, n_chunks, chunk_shift);
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

int query_val_occupancy(int* blocks) {
    int b = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, validate_kernel<true>, kValThreads, 0) != cudaSuccess)
        return -1;
    *blocks = b;
    return 0;
}

}  // namespace hetm_b200
