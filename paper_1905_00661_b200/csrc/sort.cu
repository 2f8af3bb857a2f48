// sort.cu — hand-written device primitives of the SCAN schedules (bank_sched.cu,
// cache_sched.cu): a stable LSD radix sort of (u32 key, u32 value) pairs, the
// compaction of flagged indices and the segmented {delta, last writer} scan of
// a traced bank batch.  No library kernels.
//
// Radix sort: ceil(end_bit / 8) passes of <= 8-bit digits (a 2^27-word
// shard's account keys + sentinel: 4 passes of 7 bits; 10-bit digits in 3
// passes measured slower: the per-tile look-back vector of 1024 digits is a
// quarter of the tile's payload).  One upsweep kernel counts the digits of
// every pass in one read of the keys; then ONE kernel per pass ("onesweep"):
//   * a CTA takes the next tile of kTile keys (dynamic tile ids, so earlier
//     tiles are always resident first), ranks its keys stably — each warp
//     owns a contiguous 512-key slice and ranks it with __match_any_sync —
//     and publishes the tile's per-digit counts (flag A);
//   * decoupled look-back: per digit, it walks back over the predecessors'
//     published counts (8 tiles per step, loaded at once) until a tile with an
//     inclusive prefix (flag P), then publishes its own inclusive prefix — no
//     separate scan launch, no per-tile histogram array written and re-read;
//   * the tile is staged in shared memory in digit order and written so that
//     consecutive threads store consecutive addresses of one digit's run.
// Streaming per pass: keys and values read once and written once.
#include <algorithm>

#include "common.cuh"
#include "kernels.h"

namespace hetm_b200 {

namespace {

constexpr int kSortThreads = 256;
constexpr int kSortWarps = kSortThreads / 32;
constexpr int kSortItems = 16;                          // keys per thread per tile
constexpr int kTile = kSortThreads * kSortItems;        // 4096 keys
constexpr int kSlice = kTile / kSortWarps;              // 512 keys per warp
constexpr int kMaxDigitBits = 8;
constexpr int kMaxDigits = 1 << kMaxDigitBits;
constexpr int kDigitsPerThread = kMaxDigits / kSortThreads;
constexpr int kMaxPasses = 4;                            // end_bit <= 32 at <= 8 bits per pass
// [warp][digit] counts, staged keys, staged values, tile-local digit starts, global digit bases
constexpr size_t kSweepSmem = (size_t)kSortWarps * kMaxDigits * 4 + 2 * (size_t)kTile * 4 + 2 * kMaxDigits * 4;
// look-back words: flag (2 bits) | count (62 bits)
constexpr unsigned long long kFlagA = 1ull << 62, kFlagP = 2ull << 62, kFlagMask = 3ull << 62;

__device__ __forceinline__ uint32_t digit_of(uint32_t key, int shift, uint32_t mask) { return (key >> shift) & mask; }

struct SortPasses {
    int n;
    int shift[kMaxPasses], bits[kMaxPasses];
};

// Digit totals of every pass in one read of the keys: tot[p * kMaxDigits + d].
__global__ void __launch_bounds__(kSortThreads) sort_upsweep_kernel(const uint32_t* __restrict__ keys, uint64_t n,
                                                                    SortPasses ps, uint32_t* __restrict__ tot) {
    __shared__ uint32_t h[kMaxPasses * kMaxDigits];
    for (int q = threadIdx.x; q < ps.n * kMaxDigits; q += kSortThreads) h[q] = 0;
    __syncthreads();
    for (uint64_t i = (uint64_t)blockIdx.x * kSortThreads + threadIdx.x; i < n; i += (uint64_t)gridDim.x * kSortThreads) {
        const uint32_t k = keys[i];
        for (int p = 0; p < ps.n; ++p)
            atomicAdd(&h[p * kMaxDigits + digit_of(k, ps.shift[p], (1u << ps.bits[p]) - 1)], 1u);
    }
    __syncthreads();
    for (int q = threadIdx.x; q < ps.n * kMaxDigits; q += kSortThreads)
        if (h[q]) atomicAdd(&tot[q], h[q]);
}

__global__ void __launch_bounds__(kSortThreads) sort_onesweep_kernel(const uint32_t* __restrict__ keys,
                                                                     const uint32_t* __restrict__ vals, uint64_t n,
                                                                     int shift, int bits,
                                                                     const uint32_t* __restrict__ tot,
                                                                     unsigned long long* state,
                                                                     unsigned int* tile_ctr,
                                                                     uint32_t* __restrict__ keys_out,
                                                                     uint32_t* __restrict__ vals_out) {
    extern __shared__ uint32_t sm[];
    uint32_t* cnt = sm;                                   // [warp][kMaxDigits]
    uint32_t* sk = cnt + kSortWarps * kMaxDigits;         // staged keys (tile, digit order)
    uint32_t* sv = sk + kTile;                            // staged values
    uint32_t* dstart = sv + kTile;                        // tile-local start of each digit
    uint32_t* gbase = dstart + kMaxDigits;                // global output start of each digit for this tile
    __shared__ uint32_t wpart[kSortWarps];
    __shared__ uint32_t tile_s;
    const uint32_t D = 1u << bits, mask = D - 1;
    const unsigned lane = lane_id(), w = threadIdx.x >> 5;
    if (threadIdx.x == 0) tile_s = atomicAdd(tile_ctr, 1u);
    for (uint32_t q = threadIdx.x; q < kSortWarps * kMaxDigits; q += kSortThreads) cnt[q] = 0;
    __syncthreads();
    const uint32_t tile = tile_s;
    const uint64_t t0 = (uint64_t)tile * kTile;
    const uint64_t s0 = t0 + (uint64_t)w * kSlice;  // this warp's contiguous slice
    uint32_t k[kSortItems], v[kSortItems], rk[kSortItems];
#pragma unroll
    for (int r = 0; r < kSortItems; ++r) {
        const uint64_t i = s0 + (uint64_t)r * 32 + lane;
        k[r] = i < n ? keys[i] : 0u;
        v[r] = i < n ? vals[i] : 0u;
    }
    uint32_t* wc = cnt + w * kMaxDigits;
#pragma unroll
    for (int r = 0; r < kSortItems; ++r) {
        const uint64_t i = s0 + (uint64_t)r * 32 + lane;
        const uint32_t d = i < n ? digit_of(k[r], shift, mask) : D;
        const unsigned peers = __match_any_sync(0xffffffffu, d);
        const uint32_t before = d < D ? wc[d] : 0u;
        __syncwarp();
        if (d < D && lane == (unsigned)(__ffs(peers) - 1)) wc[d] = before + __popc(peers);
        __syncwarp();
        rk[r] = before + __popc(peers & ((1u << lane) - 1u));
    }
    __syncthreads();
    // per digit (kDigitsPerThread consecutive per thread): exclusive prefix over the warps, tile count
    uint32_t tsum[kDigitsPerThread];
#pragma unroll
    for (int q = 0; q < kDigitsPerThread; ++q) {
        const uint32_t d = threadIdx.x * kDigitsPerThread + q;
        uint32_t run = 0;
        if (d < D)
            for (int ww = 0; ww < kSortWarps; ++ww) {
                const uint32_t c = cnt[ww * kMaxDigits + d];
                cnt[ww * kMaxDigits + d] = run;
                run += c;
            }
        tsum[q] = run;
    }
    // publish the tile's counts (tile 0: already inclusive)
    unsigned long long* st = state + (uint64_t)tile * kMaxDigits;
#pragma unroll
    for (int q = 0; q < kDigitsPerThread; ++q) {
        const uint32_t d = threadIdx.x * kDigitsPerThread + q;
        if (d < D) st_relaxed(&st[d], (tile == 0 ? kFlagP : kFlagA) | tsum[q]);
    }
    // global digit starts: exclusive scan of this pass's digit totals
    uint32_t my = 0, tt[kDigitsPerThread];
#pragma unroll
    for (int q = 0; q < kDigitsPerThread; ++q) {
        const uint32_t d = threadIdx.x * kDigitsPerThread + q;
        tt[q] = d < D ? tot[d] : 0u;
        my += tt[q];
    }
    uint32_t incl = my;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= (unsigned)o) incl += y;
    }
    if (lane == 31) wpart[w] = incl;
    __syncthreads();
    uint32_t gb = incl - my;
    for (unsigned q = 0; q < w; ++q) gb += wpart[q];
    // decoupled look-back per digit: + the counts of the same digit in earlier
    // tiles.  The thread's digits walk back together, kLookback predecessor
    // tiles per step (all their flag words loaded at once), so the walk to the
    // nearest inclusive prefix costs a few L2 round trips, not one per tile.
    constexpr int kLookback = 8;
    int64_t tq[kDigitsPerThread];
    unsigned long long ex[kDigitsPerThread];
    bool dn[kDigitsPerThread];
#pragma unroll
    for (int q = 0; q < kDigitsPerThread; ++q) {
        tq[q] = (int64_t)tile - 1;
        ex[q] = 0;
        dn[q] = tile == 0 || threadIdx.x * kDigitsPerThread + q >= D;
    }
    for (;;) {
        bool all = true;
#pragma unroll
        for (int q = 0; q < kDigitsPerThread; ++q) all &= dn[q];
        if (all) break;
        unsigned long long x[kDigitsPerThread][kLookback];
#pragma unroll
        for (int q = 0; q < kDigitsPerThread; ++q) {
            const uint32_t d = threadIdx.x * kDigitsPerThread + q;
#pragma unroll
            for (int j = 0; j < kLookback; ++j)
                x[q][j] = !dn[q] && tq[q] - j >= 0 ? ld_relaxed(&state[(uint64_t)(tq[q] - j) * kMaxDigits + d]) : 0ull;
        }
#pragma unroll
        for (int q = 0; q < kDigitsPerThread; ++q) {
            if (dn[q]) continue;
            int j = 0;
            for (; j < kLookback; ++j) {
                const unsigned long long y = x[q][j];
                if (!(y & kFlagMask)) break;  // that predecessor has not published yet: resume there
                ex[q] += y & ~kFlagMask;
                if (y & kFlagP) {
                    dn[q] = true;
                    break;
                }
            }
            if (!dn[q]) tq[q] -= j;
        }
    }
#pragma unroll
    for (int q = 0; q < kDigitsPerThread; ++q) {
        const uint32_t d = threadIdx.x * kDigitsPerThread + q;
        if (d < D && tile > 0) st_relaxed(&st[d], kFlagP | (ex[q] + tsum[q]));
        if (d < D) gbase[d] = gb + (uint32_t)ex[q];
        gb += tt[q];
    }
    __syncthreads();
    // block exclusive scan of the tile counts -> dstart
    my = 0;
#pragma unroll
    for (int q = 0; q < kDigitsPerThread; ++q) my += tsum[q];
    incl = my;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= (unsigned)o) incl += y;
    }
    if (lane == 31) wpart[w] = incl;
    __syncthreads();
    uint32_t base = incl - my;
    for (unsigned q = 0; q < w; ++q) base += wpart[q];
#pragma unroll
    for (int q = 0; q < kDigitsPerThread; ++q) {
        const uint32_t d = threadIdx.x * kDigitsPerThread + q;
        if (d < D) dstart[d] = base;
        base += tsum[q];
    }
    __syncthreads();
#pragma unroll
    for (int r = 0; r < kSortItems; ++r) {
        const uint64_t i = s0 + (uint64_t)r * 32 + lane;
        if (i >= n) continue;
        const uint32_t d = digit_of(k[r], shift, mask);
        const uint32_t p = dstart[d] + cnt[w * kMaxDigits + d] + rk[r];
        sk[p] = k[r];
        sv[p] = v[r];
    }
    __syncthreads();
    const uint32_t m = n - t0 < (uint64_t)kTile ? (uint32_t)(n - t0) : (uint32_t)kTile;
    for (uint32_t p = threadIdx.x; p < m; p += kSortThreads) {
        const uint32_t key = sk[p], d = digit_of(key, shift, mask);
        const uint32_t g = gbase[d] + (p - dstart[d]);
        keys_out[g] = key;
        vals_out[g] = sv[p];
    }
}

// ---- compaction of flagged indices: out = { i : flag[i] != 0 } in order
constexpr int kSelThreads = 256;
constexpr int kSelItems = 16;
constexpr int kSelTile = kSelThreads * kSelItems;

__global__ void __launch_bounds__(kSelThreads) select_count_kernel(const uint8_t* __restrict__ flag, uint64_t n,
                                                                   uint32_t* __restrict__ tile_cnt) {
    __shared__ uint32_t c;
    if (threadIdx.x == 0) c = 0;
    __syncthreads();
    const uint64_t t0 = (uint64_t)blockIdx.x * kSelTile;
    uint32_t mine = 0;
#pragma unroll
    for (int r = 0; r < kSelItems; ++r) {
        const uint64_t i = t0 + (uint64_t)r * kSelThreads + threadIdx.x;
        mine += (i < n && flag[i]) ? 1u : 0u;
    }
    mine = warp_sum(mine);
    if (lane_id() == 0 && mine) atomicAdd(&c, mine);
    __syncthreads();
    if (threadIdx.x == 0) tile_cnt[blockIdx.x] = c;
}

// One CTA: exclusive scan of the tile counts (in place) and the total.
__global__ void __launch_bounds__(1024) select_scan_kernel(uint32_t* tile_cnt, uint64_t n_tiles, uint32_t* total) {
    __shared__ uint32_t part[32];
    const unsigned lane = lane_id(), w = threadIdx.x >> 5;
    const uint64_t lo = n_tiles * threadIdx.x / 1024, hi = n_tiles * (threadIdx.x + 1) / 1024;
    uint32_t s = 0;
    for (uint64_t t = lo; t < hi; ++t) s += tile_cnt[t];
    uint32_t incl = s;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= (unsigned)o) incl += y;
    }
    if (lane == 31) part[w] = incl;
    __syncthreads();
    uint32_t run = incl - s;
    for (unsigned q = 0; q < w; ++q) run += part[q];
    for (uint64_t t = lo; t < hi; ++t) {
        const uint32_t c = tile_cnt[t];
        tile_cnt[t] = run;
        run += c;
    }
    if (threadIdx.x == 1023) *total = run;
}

// Each warp owns kSelItems consecutive 32-index groups of the tile (order:
// warp-major), so warp-local ballots + the warp prefix give stable positions.
__global__ void __launch_bounds__(kSelThreads) select_scatter_kernel(const uint8_t* __restrict__ flag, uint64_t n,
                                                                     const uint32_t* __restrict__ tile_off,
                                                                     uint32_t* __restrict__ out) {
    __shared__ uint32_t wcnt[kSelThreads / 32];
    const unsigned lane = lane_id(), w = threadIdx.x >> 5;
    const uint64_t s0 = (uint64_t)blockIdx.x * kSelTile + (uint64_t)w * (kSelItems * 32);
    unsigned m[kSelItems];
    uint32_t c = 0;
#pragma unroll
    for (int r = 0; r < kSelItems; ++r) {
        const uint64_t i = s0 + (uint64_t)r * 32 + lane;
        m[r] = __ballot_sync(0xffffffffu, i < n && flag[i]);
        c += __popc(m[r]);
    }
    if (lane == 0) wcnt[w] = c;
    __syncthreads();
    uint32_t pos = tile_off[blockIdx.x];
    for (unsigned q = 0; q < w; ++q) pos += wcnt[q];
#pragma unroll
    for (int r = 0; r < kSelItems; ++r) {
        if ((m[r] >> lane) & 1u) out[pos + __popc(m[r] & ((1u << lane) - 1u))] = (uint32_t)(s0 + (uint64_t)r * 32 + lane);
        pos += __popc(m[r]);
    }
}

// ---- segmented inclusive scan of {delta, last writer} by key (traced bank SCAN)
constexpr int kSegThreads = 256;
constexpr int kSegItems = 16;
constexpr int kSegTile = kSegThreads * kSegItems;

struct SegVal {
    unsigned long long d, w;  // summed delta, last writer (kNoWriter: none)
};
constexpr unsigned long long kNoWriter = ~0ull;
__device__ __forceinline__ SegVal seg_op(SegVal a, SegVal b) { return SegVal{a.d + b.d, b.w != kNoWriter ? b.w : a.w}; }

// value of sorted access j: its delta (indexed by access) and, when it is the
// writer slot, its transaction (payload layout of bank_sched.cu, S = 4)
__device__ __forceinline__ SegVal seg_value(const uint32_t* pay, const unsigned long long* delta, uint64_t j) {
    const uint32_t p = pay[j];
    return SegVal{delta[p >> 1], (p & 1u) ? (unsigned long long)(p >> 3) : kNoWriter};
}

// Per tile: the aggregate of the elements after (and including) its last
// segment head, and whether it has a head.
__global__ void __launch_bounds__(kSegThreads) seg_tile_kernel(const uint32_t* __restrict__ keys,
                                                               const uint32_t* __restrict__ pay,
                                                               const unsigned long long* __restrict__ delta,
                                                               uint64_t n, SegVal* __restrict__ agg,
                                                               uint32_t* __restrict__ has_head) {
    __shared__ SegVal ta[kSegThreads];
    __shared__ uint32_t th[kSegThreads];
    const uint64_t t0 = (uint64_t)blockIdx.x * kSegTile, b = t0 + (uint64_t)threadIdx.x * kSegItems;
    SegVal acc{0, kNoWriter};
    uint32_t head = 0;
    for (int r = 0; r < kSegItems; ++r) {
        const uint64_t j = b + r;
        if (j >= n) break;
        const bool h = j == 0 || keys[j] != keys[j - 1];
        const SegVal x = seg_value(pay, delta, j);
        acc = h ? x : seg_op(acc, x);
        head |= h;
    }
    ta[threadIdx.x] = acc;
    th[threadIdx.x] = head;
    __syncthreads();
    if (threadIdx.x == 0) {  // fold the threads' suffix aggregates in order
        SegVal a{0, kNoWriter};
        uint32_t hh = 0;
        for (int q = 0; q < kSegThreads; ++q) {
            a = th[q] ? ta[q] : seg_op(a, ta[q]);
            hh |= th[q];
        }
        agg[blockIdx.x] = a;
        has_head[blockIdx.x] = hh;
    }
}

// Carry into every tile (one thread: traced batches only).
__global__ void seg_carry_kernel(const SegVal* agg, const uint32_t* has_head, uint64_t n_tiles, SegVal* carry) {
    SegVal c{0, kNoWriter};
    for (uint64_t t = 0; t < n_tiles; ++t) {
        carry[t] = c;
        c = has_head[t] ? agg[t] : seg_op(c, agg[t]);
    }
}

__global__ void __launch_bounds__(kSegThreads) seg_scan_kernel(const uint32_t* __restrict__ keys,
                                                               const uint32_t* __restrict__ pay,
                                                               const unsigned long long* __restrict__ delta,
                                                               uint64_t n, const SegVal* __restrict__ carry,
                                                               unsigned long long* __restrict__ out) {
    __shared__ SegVal ta[kSegThreads];
    __shared__ uint32_t th[kSegThreads];
    const uint64_t t0 = (uint64_t)blockIdx.x * kSegTile, b = t0 + (uint64_t)threadIdx.x * kSegItems;
    SegVal acc{0, kNoWriter};
    uint32_t head = 0;
    for (int r = 0; r < kSegItems; ++r) {
        const uint64_t j = b + r;
        if (j >= n) break;
        const bool h = j == 0 || keys[j] != keys[j - 1];
        const SegVal x = seg_value(pay, delta, j);
        acc = h ? x : seg_op(acc, x);
        head |= h;
    }
    ta[threadIdx.x] = acc;
    th[threadIdx.x] = head;
    __syncthreads();
    if (threadIdx.x == 0) {  // exclusive carry into every thread, in order, from the tile's carry-in
        SegVal c = carry[blockIdx.x];
        for (int q = 0; q < kSegThreads; ++q) {
            const SegVal a = ta[q];
            const uint32_t h = th[q];
            ta[q] = c;
            c = h ? a : seg_op(c, a);
        }
    }
    __syncthreads();
    SegVal c = ta[threadIdx.x];
    for (int r = 0; r < kSegItems; ++r) {
        const uint64_t j = b + r;
        if (j >= n) break;
        const bool h = j == 0 || keys[j] != keys[j - 1];
        const SegVal x = seg_value(pay, delta, j);
        c = h ? x : seg_op(c, x);
        out[2 * j] = c.d;
        out[2 * j + 1] = c.w;
    }
}

int digit_passes(int end_bit) { return end_bit <= 0 ? 0 : (end_bit + kMaxDigitBits - 1) / kMaxDigitBits; }
size_t al256(size_t x) { return (x + 255) & ~size_t(255); }

}  // namespace

cudaError_t radix_sort_init() {
    static const cudaError_t attr = cudaFuncSetAttribute(sort_onesweep_kernel,
                                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSweepSmem);
    return attr;
}

size_t radix_sort_temp_bytes(uint64_t n, int end_bit) {
    const uint64_t tiles = (n + kTile - 1) / kTile;
    const int P = digit_passes(end_bit);
    // [tmp keys | tmp vals | digit totals per pass | tile counters | look-back words per pass]
    return 2 * al256(n * 4) + al256(kMaxPasses * kMaxDigits * 4) + 256 +
           al256((size_t)std::max(P, 1) * tiles * kMaxDigits * 8);
}

cudaError_t radix_sort_pairs(const uint32_t* keys_in, uint32_t* keys_out, const uint32_t* vals_in, uint32_t* vals_out,
                             uint64_t n, int end_bit, void* temp, size_t temp_bytes, const LaunchGeom& g, cudaStream_t s) {
    if (n == 0) return cudaSuccess;
    if (n >= (1ull << 32) || end_bit > 32 || temp_bytes < radix_sort_temp_bytes(n, end_bit))
        return cudaErrorInvalidValue;
    const int P = digit_passes(end_bit);
    if (P == 0) {
        cudaError_t e = cudaMemcpyAsync(keys_out, keys_in, n * 4, cudaMemcpyDeviceToDevice, s);
        return e == cudaSuccess ? cudaMemcpyAsync(vals_out, vals_in, n * 4, cudaMemcpyDeviceToDevice, s) : e;
    }
    if (cudaError_t e = radix_sort_init(); e != cudaSuccess) return e;
    const uint64_t tiles = (n + kTile - 1) / kTile;
    char* p = static_cast<char*>(temp);
    uint32_t* tk = reinterpret_cast<uint32_t*>(p);
    uint32_t* tv = reinterpret_cast<uint32_t*>(p + al256(n * 4));
    char* meta = p + 2 * al256(n * 4);
    uint32_t* tot = reinterpret_cast<uint32_t*>(meta);
    unsigned int* tile_ctr = reinterpret_cast<unsigned int*>(meta + al256(kMaxPasses * kMaxDigits * 4));
    auto* state = reinterpret_cast<unsigned long long*>(meta + al256(kMaxPasses * kMaxDigits * 4) + 256);
    const size_t meta_bytes = al256(kMaxPasses * kMaxDigits * 4) + 256 + (size_t)P * tiles * kMaxDigits * 8;
    cudaError_t e = cudaMemsetAsync(meta, 0, meta_bytes, s);  // totals, tile counters, look-back flags
    if (e != cudaSuccess) return e;
    SortPasses ps{};
    ps.n = P;
    const int per = (end_bit + P - 1) / P;  // balanced digit widths
    for (int q = 0, shift = 0; q < P; ++q) {
        ps.shift[q] = shift;
        ps.bits[q] = std::min(per, end_bit - shift);
        shift += ps.bits[q];
    }
    const uint64_t want = (n + kSortThreads * 16 - 1) / (kSortThreads * 16);
    const unsigned ugrid = (unsigned)std::max<uint64_t>(1, std::min<uint64_t>(want, (uint64_t)g.sm_count * 4));
    sort_upsweep_kernel<<<ugrid, kSortThreads, 0, s>>>(keys_in, n, ps, tot);
    const uint32_t* src_k = keys_in;
    const uint32_t* src_v = vals_in;
    for (int q = 0; q < P; ++q) {
        // the last pass writes the output; earlier ones alternate so that holds
        const bool to_out = ((P - 1 - q) & 1) == 0;
        uint32_t* dk = to_out ? keys_out : tk;
        uint32_t* dv = to_out ? vals_out : tv;
        sort_onesweep_kernel<<<(unsigned)tiles, kSortThreads, kSweepSmem, s>>>(
            src_k, src_v, n, ps.shift[q], ps.bits[q], tot + q * kMaxDigits, state + (uint64_t)q * tiles * kMaxDigits,
            tile_ctr + q, dk, dv);
        src_k = dk;
        src_v = dv;
    }
    return cudaGetLastError();
}

size_t select_flagged_temp_bytes(uint64_t n) { return al256(((n + kSelTile - 1) / kSelTile) * 4); }

cudaError_t select_flagged(const uint8_t* flags, uint64_t n, uint32_t* out, uint32_t* d_count, void* temp,
                           size_t temp_bytes, cudaStream_t s) {
    if (n == 0) return cudaMemsetAsync(d_count, 0, 4, s);
    if (n >= (1ull << 32) || temp_bytes < select_flagged_temp_bytes(n)) return cudaErrorInvalidValue;
    const uint64_t tiles = (n + kSelTile - 1) / kSelTile;
    auto* tc = static_cast<uint32_t*>(temp);
    select_count_kernel<<<(unsigned)tiles, kSelThreads, 0, s>>>(flags, n, tc);
    select_scan_kernel<<<1, 1024, 0, s>>>(tc, tiles, d_count);
    select_scatter_kernel<<<(unsigned)tiles, kSelThreads, 0, s>>>(flags, n, tc, out);
    return cudaGetLastError();
}

size_t seg_scan_temp_bytes(uint64_t n) {
    const uint64_t tiles = (n + kSegTile - 1) / kSegTile;
    return 2 * al256(tiles * sizeof(SegVal)) + al256(tiles * 4);
}

cudaError_t seg_scan_delta_writer(const uint32_t* keys, const uint32_t* pay, const unsigned long long* delta,
                                  uint64_t n, unsigned long long* out, void* temp, size_t temp_bytes, cudaStream_t s) {
    if (n == 0) return cudaSuccess;
    if (temp_bytes < seg_scan_temp_bytes(n)) return cudaErrorInvalidValue;
    const uint64_t tiles = (n + kSegTile - 1) / kSegTile;
    char* p = static_cast<char*>(temp);
    auto* agg = reinterpret_cast<SegVal*>(p);
    auto* carry = reinterpret_cast<SegVal*>(p + al256(tiles * sizeof(SegVal)));
    auto* hh = reinterpret_cast<uint32_t*>(p + 2 * al256(tiles * sizeof(SegVal)));
    seg_tile_kernel<<<(unsigned)tiles, kSegThreads, 0, s>>>(keys, pay, delta, n, agg, hh);
    seg_carry_kernel<<<1, 1, 0, s>>>(agg, hh, tiles, carry);
    seg_scan_kernel<<<(unsigned)tiles, kSegThreads, 0, s>>>(keys, pay, delta, n, carry, out);
    return cudaGetLastError();
}

}  // namespace hetm_b200
