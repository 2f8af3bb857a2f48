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

template <bool kApply>
__global__ void __launch_bounds__(kValThreads) validate_kernel(ShardView v, const hetm_log_entry* __restrict__ log,
                                                               uint64_t n, uint64_t ts_floor, DevCounters* ctr) {
    unsigned conflict = 0, bad = 0, oob = 0;
    unsigned long long maxts = 0;
    const uint64_t span = (uint64_t)gridDim.x * blockDim.x * kUnroll;
    for (uint64_t i0 = (uint64_t)blockIdx.x * blockDim.x * kUnroll + threadIdx.x; i0 < n; i0 += span) {
        EntryRegs e[kUnroll];
#pragma unroll
        for (int u = 0; u < kUnroll; ++u) {
            const uint64_t i = i0 + (uint64_t)u * blockDim.x;
            e[u] = i < n ? load_entry(log, i) : EntryRegs{v.base, 0, ~0ull};
        }
#pragma unroll
        for (int u = 0; u < kUnroll; ++u) {
            if (i0 + (uint64_t)u * blockDim.x >= n) continue;
            const uint64_t loc = e[u].addr - v.base;
            if (loc >= v.size_words) {
                oob = 1;
                continue;
            }
            const uint64_t bit = loc >> v.gran_shift;
            conflict |= (unsigned)((v.rs[bit >> 6] >> (bit & 63)) & 1ull);  // (a) RS test
            bad |= (e[u].ts <= ts_floor);
            maxts = e[u].ts > maxts ? e[u].ts : maxts;
            if (kApply) atomicMax(&v.cells[loc].ts, (unsigned long long)e[u].ts);  // (b) pass A
        }
    }
    conflict = __any_sync(0xffffffffu, conflict);
    bad = __any_sync(0xffffffffu, bad);
    oob = __any_sync(0xffffffffu, oob);
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

// Pass B (dst == nullptr: into the cells' value field) and its variants for
// the shadow patch / rollback (dst = plain word array): the entry whose ts
// equals the cell's TS is the freshest one for that word.
__global__ void __launch_bounds__(kValThreads) winner_kernel(Cell* cells, uint64_t* dst, uint64_t base,
                                                             uint64_t size_words, const hetm_log_entry* __restrict__ log,
                                                             uint64_t n) {
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
            cur[u] = loc < size_words ? ld_relaxed(&cells[loc].ts) : ~0ull;
        }
#pragma unroll
        for (int u = 0; u < kUnroll; ++u) {
            if (cur[u] != e[u].ts) continue;
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

static unsigned grid_cap(uint64_t items, int threads, const LaunchGeom& g, int per_sm) {
    uint64_t want = (items + threads - 1) / threads;
    const uint64_t cap = (uint64_t)per_sm * (uint64_t)g.sm_count;
    if (want > cap) want = cap;
    return (unsigned)(want ? want : 1);
}

cudaError_t launch_validate(const ShardView& v, const hetm_log_entry* d_log, uint64_t n, int apply, uint64_t ts_floor,
                            DevCounters* ctr, const LaunchGeom& g, cudaStream_t s) {
    if (n == 0) return cudaSuccess;
    const unsigned grid = grid_cap((n + kUnroll - 1) / kUnroll, kValThreads, g, g.max_blocks_val);
    if (apply) {
        validate_kernel<true><<<grid, kValThreads, 0, s>>>(v, d_log, n, ts_floor, ctr);
        winner_kernel<<<grid, kValThreads, 0, s>>>(v.cells, nullptr, v.base, v.size_words, d_log, n);
    } else {
        validate_kernel<false><<<grid, kValThreads, 0, s>>>(v, d_log, n, ts_floor, ctr);
    }
    return cudaGetLastError();
}

cudaError_t launch_winner_apply(Cell* cells, uint64_t* dst, uint64_t base, uint64_t size_words,
                                const hetm_log_entry* d_log, uint64_t n, const LaunchGeom& g, cudaStream_t s) {
    if (n == 0) return cudaSuccess;
    const unsigned grid = grid_cap((n + kUnroll - 1) / kUnroll, kValThreads, g, g.max_blocks_val);
    winner_kernel<<<grid, kValThreads, 0, s>>>(cells, dst, base, size_words, d_log, n);
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
