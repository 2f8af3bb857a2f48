// cells.cu — conversions between the 32-B word-cell layout of devReplica
// (common.cuh) and plain 64-bit word arrays (devShadow, raw-op staging).
// Used at the edges only: raw ops, the shadow refresh of
// mergeCommit and the rollback of mergeAbortDevice.
#include <cstdlib>

#include "common.cuh"
#include "kernels.h"

namespace hetm_b200 {

// dst[i] = cells[lo + i].value
__global__ void gather_range_kernel(uint64_t* __restrict__ dst, const Cell* __restrict__ cells, uint64_t lo, uint64_t n) {
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
        dst[i] = cells[lo + i].value;
}

// cells[lo + i].value = src[i]
__global__ void scatter_range_kernel(Cell* __restrict__ cells, const uint64_t* __restrict__ src, uint64_t lo, uint64_t n) {
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
        cells[lo + i].value = src[i];
}

// For every dirty chunk c: plain[w] <-> cells[w].value for w in chunk c.
// One CTA walks one dirty chunk at a time (grid-stride over chunks).
template <bool kToPlain>
__global__ void dirty_chunks_kernel(uint64_t* __restrict__ plain, Cell* __restrict__ cells, uint64_t size_words,
                                    const unsigned long long* __restrict__ bits, uint64_t n_chunks,
                                    uint32_t chunk_shift) {
    const uint64_t wpc = 1ull << chunk_shift;
    for (uint64_t c = blockIdx.x; c < n_chunks; c += gridDim.x) {
        if (bits && !((bits[c >> 6] >> (c & 63)) & 1ull)) continue;
        const uint64_t lo = c * wpc;
        const uint64_t hi = lo + wpc < size_words ? lo + wpc : size_words;
        for (uint64_t w = lo + threadIdx.x; w < hi; w += blockDim.x) {
            if (kToPlain) plain[w] = cells[w].value;
            else cells[w].value = plain[w];
        }
    }
}

// mergeCommit delta, step 1 of 2 (replaces a radix sort of the log): every
// write-set log slot claims its word in a W-bit claim bitmap (one returning
// atomicOr into L2-resident words); the first claimer of a word appends it to
// the unique-word list (warp-aggregated) and counts it in its address bucket
// (kDeltaBuckets contiguous word ranges, per-CTA shared histogram).  The
// write-set log itself is left untouched (the rollback reads it).
constexpr int kClaimThreads = 256;
// gate != nullptr (a merge staged before the host has read the verdict): the
// slot count comes from the device counters and nothing is staged when the
// round has a conflict or its write-set log overflowed.
__global__ void __launch_bounds__(kClaimThreads) delta_claim_kernel(const uint32_t* __restrict__ wlog, uint64_t n,
                                                                    uint64_t size_words, unsigned long long* claim,
                                                                    uint32_t* __restrict__ uniq,
                                                                    unsigned long long* n_uniq, uint32_t* bucket_cnt,
                                                                    uint32_t bshift, const DevCounters* gate) {
    __shared__ uint32_t hist[kDeltaBuckets];
    if (gate) {
        if (gate->conflict || gate->wlog_overflow) return;
        const uint64_t used = 2 * (gate->ticket - gate->wlog_base);
        n = used < n ? used : n;
    }
    for (int b = threadIdx.x; b < kDeltaBuckets; b += blockDim.x) hist[b] = 0;
    __syncthreads();
    const unsigned lane = lane_id();
    const uint64_t warp = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const uint64_t warps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    for (uint64_t base = warp * 32; base < n; base += warps * 32) {  // warp-uniform trip count
        const uint64_t i = base + lane;
        const uint32_t loc = i < n ? wlog[i] : ~0u;
        bool first = false;
        if (loc < size_words) {
            const unsigned long long m = 1ull << (loc & 63);
            first = !(atomicOr(&claim[loc >> 6], m) & m);
        }
        const unsigned ballot = __ballot_sync(0xffffffffu, first);
        if (!ballot) continue;
        unsigned long long at = 0;
        if (lane == (unsigned)(__ffs(ballot) - 1)) at = atomicAdd(n_uniq, (unsigned long long)__popc(ballot));
        at = __shfl_sync(0xffffffffu, at, __ffs(ballot) - 1);
        if (first) {
            uniq[at + __popc(ballot & ((1u << lane) - 1))] = loc;
            atomicAdd(&hist[loc >> bshift], 1u);
        }
    }
    __syncthreads();
    for (int b = threadIdx.x; b < kDeltaBuckets; b += blockDim.x)
        if (hist[b]) atomicAdd(&bucket_cnt[b], hist[b]);
}

// Step 1, versioned form (rounds whose batches all commit with per-word
// versions: bank and rw kernels, both schedules): no claim bitmap.  A word's
// cell carries the commit version of its LAST writer of the round (ticket + 1,
// device_tm.cuh lk_commit), and the write-set log slot of ticket t is
// 2 (t - wlog_base) + j, so exactly one slot per written word sees
// meta == version(its own ticket) — that slot picks the word and the value it
// read with the same 16-B load.  (A host-log apply retags a word's meta only
// in a conflicting round, which is never merged.)  The second slot of a
// transaction repeating its first word is skipped.  Output is slot-indexed
// (ploc[s] = the word or ~0u, pval[s] = its value: coalesced stores, no
// compaction atomics); the record count and slot count go to n_out[0..1].
__global__ void __launch_bounds__(kClaimThreads) delta_pick_kernel(const uint32_t* __restrict__ wlog, uint64_t n,
                                                                   uint64_t size_words, const Cell* __restrict__ cells,
                                                                   uint32_t* __restrict__ ploc,
                                                                   uint64_t* __restrict__ pval,
                                                                   unsigned long long* n_out, uint32_t* bucket_cnt,
                                                                   uint32_t bshift, const DevCounters* ctr, int gated) {
    __shared__ uint32_t hist[kDeltaBuckets];
    __shared__ uint32_t picked;
    if (gated) {
        if (ctr->conflict || ctr->wlog_overflow) n = 0;  // nothing is staged: emit sees 0 slots
        const uint64_t used = 2 * (ctr->ticket - ctr->wlog_base);
        n = used < n ? used : n;
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) n_out[1] = n;
    if (n == 0) return;
    const unsigned long long wbase = ctr->wlog_base;
    for (int b = threadIdx.x; b < kDeltaBuckets; b += blockDim.x) hist[b] = 0;
    if (threadIdx.x == 0) picked = 0;
    __syncthreads();
    const unsigned lane = lane_id();
    const uint64_t warp = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const uint64_t warps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    uint32_t mine = 0;
    for (uint64_t base = warp * 32; base < n; base += warps * 32) {  // warp-uniform trip count; slot pairs in one warp
        const uint64_t i = base + lane;
        const uint32_t loc = i < n ? wlog[i] : ~0u;
        const uint32_t prev = __shfl_up_sync(0xffffffffu, loc, 1);
        bool pick = false;
        uint64_t val = 0;
        if (loc < size_words && !((i & 1) && prev == loc)) {
            const ulonglong2 c = *reinterpret_cast<const ulonglong2*>(&cells[loc]);  // {value, meta}
            pick = c.y == ((wbase + (i >> 1) + 1) & 0x7fffffffull);
            val = c.x;
        }
        if (i < n) {
            ploc[i] = pick ? loc : ~0u;
            pval[i] = val;
        }
        if (pick) {
            atomicAdd(&hist[loc >> bshift], 1u);
            ++mine;
        }
    }
    atomicAdd(&picked, mine);
    __syncthreads();
    for (int b = threadIdx.x; b < kDeltaBuckets; b += blockDim.x)
        if (hist[b]) atomicAdd(&bucket_cnt[b], hist[b]);
    if (threadIdx.x == 0 && picked) atomicAdd(&n_out[0], (unsigned long long)picked);
}

// Step 2: each unique word becomes one {word, value} record in its address
// bucket's range (kDeltaBuckets contiguous word ranges), so the delta reaches
// the host grouped by address — a host worker's block of records covers one
// slice of the replica — and each word appears once (the speculative
// swap/undo of hetm_dev_merge_prepare needs that).  A CTA partitions a tile
// of kEmitTile records in shared memory (counting sort by bucket) and
// reserves one run per (tile, bucket) with a single global atomic, so the
// record stores land as contiguous runs instead of one scattered store per
// record.  The same value refreshes devShadow; after a claim pass the claim
// words are cleared for the next stage.
// records per thread per tile: 8 (2048-record tiles, 1024 CTAs per 2^21
// slots) beat 16 by ~10 us per cfg2 round (profiles/r02am_emit_sweep.txt)
constexpr int kEmitPer = 8;
static_assert(kDeltaBuckets == kClaimThreads, "one bucket per thread in the emit scans");
template <int PER>
__global__ void __launch_bounds__(kClaimThreads) delta_emit_kernel(const uint32_t* __restrict__ uniq,
                                                                   const unsigned long long* n_in,
                                                                   const uint32_t* __restrict__ bucket_cnt,
                                                                   uint32_t* cursor, uint32_t bshift,
                                                                   const Cell* __restrict__ cells,
                                                                   const uint64_t* __restrict__ uniq_val, DeltaBuf out,
                                                                   uint64_t* __restrict__ shadow,
                                                                   unsigned long long* claim) {
    __shared__ uint32_t first[kDeltaBuckets];  // global start of each bucket's range
    __shared__ uint32_t cnt[kDeltaBuckets];    // tile histogram, then the tile's local cursors
    __shared__ uint32_t run[kDeltaBuckets];    // global start of the tile's run in each bucket
    __shared__ uint32_t wsum[kClaimThreads / 32];
    const unsigned t = threadIdx.x, lane = lane_id(), wid = t >> 5;
    {  // exclusive scan of the bucket counts (one per thread)
        const uint32_t c = bucket_cnt[t];
        uint32_t x = c;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
            if (lane >= (unsigned)o) x += y;
        }
        if (lane == 31) wsum[wid] = x;
        __syncthreads();
        uint32_t off = 0;
        for (unsigned w = 0; w < wid; ++w) off += wsum[w];
        first[t] = off + x - c;
    }
    const uint64_t n = *n_in;  // unique words (claim pass) or slots (pick pass: ~0u = not picked)
    for (uint64_t t0 = (uint64_t)blockIdx.x * ((uint64_t)kClaimThreads * PER); t0 < n; t0 += (uint64_t)gridDim.x * ((uint64_t)kClaimThreads * PER)) {
        cnt[t] = 0;
        __syncthreads();
        uint32_t loc[PER], r[PER];
        uint64_t val[PER];
#pragma unroll
        for (int k = 0; k < PER; ++k) {
            const uint64_t j = t0 + (uint64_t)k * kClaimThreads + t;
            loc[k] = j < n ? uniq[j] : ~0u;
            val[k] = loc[k] != ~0u ? (uniq_val ? uniq_val[j] : cells[loc[k]].value) : 0;  // pick: read already
        }
#pragma unroll
        for (int k = 0; k < PER; ++k)
            if (loc[k] != ~0u) r[k] = atomicAdd(&cnt[loc[k] >> bshift], 1u);
        __syncthreads();
        if (cnt[t]) run[t] = first[t] + atomicAdd(&cursor[t], cnt[t]);
        __syncthreads();
#pragma unroll
        for (int k = 0; k < PER; ++k) {
            if (loc[k] == ~0u) continue;
            const uint32_t pos = run[loc[k] >> bshift] + r[k];
            out.loc[pos] = loc[k];
            out.val[pos] = val[k];
            if (shadow) shadow[loc[k]] = val[k];
            if (!uniq_val) claim[loc[k] >> 6] = 0;
        }
        __syncthreads();  // cnt / run are reused by the next tile
    }
}

// devShadow refresh from staged delta records (a prepared merge).
__global__ void delta_to_shadow_kernel(uint64_t* __restrict__ shadow, DeltaBuf d, uint64_t n) {
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t loc = d.loc[i];
        if (loc != ~0u) shadow[loc] = d.val[i];
    }
}

// Rollback: cells[loc].value = shadow[loc] for every write-set log slot.
__global__ void wlog_restore_kernel(Cell* __restrict__ cells, const uint64_t* __restrict__ shadow,
                                    const uint32_t* __restrict__ wlog, uint64_t n, uint64_t size_words) {
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t loc = wlog[i];
        if (loc < size_words) cells[loc].value = shadow[loc];
    }
}

// The first part of the sorted delta goes straight into the (mapped, pinned)
// host replica as zero-copy PCIe stores, concurrently with the DMA + host
// scatter of the rest.
__global__ void delta_zc_scatter_kernel(uint64_t* host, DeltaBuf d, uint64_t n) {
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t loc = d.loc[i];
        if (loc != ~0u) host[loc] = d.val[i];
    }
}

static unsigned grid_words(uint64_t n, const LaunchGeom& g) {
    uint64_t want = (n + 255) / 256;
    const uint64_t cap = (uint64_t)g.sm_count * 16;
    return (unsigned)(want < 1 ? 1 : (want > cap ? cap : want));
}

cudaError_t launch_gather_range(uint64_t* dst, const Cell* cells, uint64_t lo, uint64_t n, const LaunchGeom& g,
                                cudaStream_t s) {
    if (n == 0) return cudaSuccess;
    gather_range_kernel<<<grid_words(n, g), 256, 0, s>>>(dst, cells, lo, n);
    return cudaGetLastError();
}

cudaError_t launch_scatter_range(Cell* cells, const uint64_t* src, uint64_t lo, uint64_t n, const LaunchGeom& g,
                                 cudaStream_t s) {
    if (n == 0) return cudaSuccess;
    scatter_range_kernel<<<grid_words(n, g), 256, 0, s>>>(cells, src, lo, n);
    return cudaGetLastError();
}

cudaError_t launch_delta_to_shadow(uint64_t* shadow, DeltaBuf d, uint64_t n, const LaunchGeom& g, cudaStream_t s) {
    if (n == 0) return cudaSuccess;
    delta_to_shadow_kernel<<<grid_words(n, g), 256, 0, s>>>(shadow, d, n);
    return cudaGetLastError();
}

static uint32_t word_bits(uint64_t size_words) {
    uint32_t b = 1;
    while (b < 32 && (1ull << b) < size_words) ++b;
    return b;
}

uint32_t delta_bucket_shift(uint64_t size_words) {
    const uint32_t b = word_bits(size_words);
    return b > kDeltaBucketBits ? b - kDeltaBucketBits : 0;
}

// n_uniq[0..1] and the bucket counts/cursors: one memset when contiguous.
static cudaError_t clear_stage_counters(const DeltaScratch& ds, cudaStream_t s) {
    if (ds.counters_bytes) return cudaMemsetAsync(ds.n_uniq, 0, ds.counters_bytes, s);
    cudaError_t e = cudaMemsetAsync(ds.n_uniq, 0, 2 * sizeof(unsigned long long), s);
    if (e == cudaSuccess) e = cudaMemsetAsync(ds.bucket_cnt, 0, 2 * kDeltaBuckets * sizeof(uint32_t), s);
    return e;
}

cudaError_t launch_delta_claim(const uint32_t* wlog, uint64_t n, uint64_t size_words, const DeltaScratch& ds,
                               const LaunchGeom& g, cudaStream_t s, const DevCounters* gate) {
    cudaError_t e = clear_stage_counters(ds, s);
    if (e != cudaSuccess || n == 0) return e;
    uint64_t want = (n + kClaimThreads - 1) / kClaimThreads;
    const uint64_t cap = (uint64_t)g.sm_count * 8;
    delta_claim_kernel<<<(unsigned)(want < cap ? want : cap), kClaimThreads, 0, s>>>(
        wlog, n, size_words, ds.claim, ds.uniq, ds.n_uniq, ds.bucket_cnt, delta_bucket_shift(size_words), gate);
    return cudaGetLastError();
}

cudaError_t launch_delta_pick(const uint32_t* wlog, uint64_t n, uint64_t size_words, const Cell* cells,
                              const DeltaScratch& ds, const LaunchGeom& g, cudaStream_t s, const DevCounters* ctr,
                              bool gated) {
    cudaError_t e = clear_stage_counters(ds, s);
    if (e != cudaSuccess || n == 0) return e;
    uint64_t want = (n + kClaimThreads - 1) / kClaimThreads;
    const uint64_t cap = (uint64_t)g.sm_count * 8;
    delta_pick_kernel<<<(unsigned)(want < cap ? want : cap), kClaimThreads, 0, s>>>(
        wlog, n, size_words, cells, ds.uniq, ds.uniq_val, ds.n_uniq, ds.bucket_cnt, delta_bucket_shift(size_words),
        ctr, gated ? 1 : 0);  // n_uniq[0] = records, n_uniq[1] = slots
    return cudaGetLastError();
}

cudaError_t launch_delta_emit(uint64_t max_records, uint64_t size_words, const DeltaScratch& ds, const Cell* cells,
                              DeltaBuf out, uint64_t* shadow, const LaunchGeom& g, cudaStream_t s, bool picked) {
    if (max_records == 0) return cudaSuccess;
    static const int per = [] {  // tuning experiments: HETM_EMIT_PER (4, 8 or 16 records per thread per tile)
        const char* e = std::getenv("HETM_EMIT_PER");
        const int v = e ? std::atoi(e) : kEmitPer;
        return v == 4 || v == 16 ? v : kEmitPer;
    }();
    static const uint64_t ctas = [] {  // tuning experiments: HETM_EMIT_CTAS resident CTAs per SM
        const char* e = std::getenv("HETM_EMIT_CTAS");
        return e ? (uint64_t)std::atoi(e) : 4ull;
    }();
    const uint64_t tile = (uint64_t)kClaimThreads * per;
    uint64_t want = (max_records + tile - 1) / tile;
    const uint64_t cap = (uint64_t)g.sm_count * (ctas ? ctas : 4);
    const unsigned grid = (unsigned)(want < cap ? want : cap);
    if (per == 4)
        delta_emit_kernel<4><<<grid, kClaimThreads, 0, s>>>(
            ds.uniq, picked ? ds.n_uniq + 1 : ds.n_uniq, ds.bucket_cnt, ds.bucket_cnt + kDeltaBuckets,
            delta_bucket_shift(size_words), cells, picked ? ds.uniq_val : nullptr, out, shadow, ds.claim);
    else if (per == 16)
        delta_emit_kernel<16><<<grid, kClaimThreads, 0, s>>>(
            ds.uniq, picked ? ds.n_uniq + 1 : ds.n_uniq, ds.bucket_cnt, ds.bucket_cnt + kDeltaBuckets,
            delta_bucket_shift(size_words), cells, picked ? ds.uniq_val : nullptr, out, shadow, ds.claim);
    else
        delta_emit_kernel<kEmitPer><<<grid, kClaimThreads, 0, s>>>(
            ds.uniq, picked ? ds.n_uniq + 1 : ds.n_uniq, ds.bucket_cnt, ds.bucket_cnt + kDeltaBuckets,
            delta_bucket_shift(size_words), cells, picked ? ds.uniq_val : nullptr, out, shadow, ds.claim);
    return cudaGetLastError();
}

cudaError_t launch_wlog_restore(Cell* cells, const uint64_t* shadow, const uint32_t* wlog, uint64_t n,
                                uint64_t size_words, const LaunchGeom& g, cudaStream_t s) {
    if (n == 0) return cudaSuccess;
    wlog_restore_kernel<<<grid_words(n, g), 256, 0, s>>>(cells, shadow, wlog, n, size_words);
    return cudaGetLastError();
}

cudaError_t launch_delta_zc_scatter(uint64_t* host_dev, DeltaBuf d, uint64_t n, const LaunchGeom& g,
                                    cudaStream_t s) {
    if (n == 0) return cudaSuccess;
    static const int zc_blocks = [] {  // tuning experiments only: CTAs of 128 threads per SM
        const char* e = std::getenv("HETM_ZC_BLOCKS_PER_SM");
        return e ? std::atoi(e) : 1;
    }();
    delta_zc_scatter_kernel<<<(unsigned)(g.sm_count * (zc_blocks > 0 ? zc_blocks : 1)), 128, 0, s>>>(host_dev, d, n);
    return cudaGetLastError();
}

cudaError_t launch_dirty_chunks(uint64_t* plain, Cell* cells, uint64_t size_words, const unsigned long long* bits,
                                uint64_t n_chunks, uint32_t chunk_shift, bool to_plain, const LaunchGeom& g,
                                cudaStream_t s) {
    if (n_chunks == 0) return cudaSuccess;
    const uint64_t cap = (uint64_t)g.sm_count * 8;
    const unsigned grid = (unsigned)(n_chunks < cap ? n_chunks : cap);
    if (to_plain) dirty_chunks_kernel<true><<<grid, 256, 0, s>>>(plain, cells, size_words, bits, n_chunks, chunk_shift);
    else dirty_chunks_kernel<false><<<grid, 256, 0, s>>>(plain, cells, size_words, bits, n_chunks, chunk_shift);
    return cudaGetLastError();
}

}  // namespace hetm_b200
