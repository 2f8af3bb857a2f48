// route.cu — shard router for address-range sharded validation.
//
// Shard s owns global words [s*shard_words, (s+1)*shard_words).  The router
// stable-partitions a log buffer by owner shard so the buckets can be sent
// all-to-all (NCCL over NVLink) and validated/applied locally by the owner.
//
// Warp-granular counting sort, no block-level barriers on the data path:
//   1. count   — every warp owns a contiguous slice of the log and counts its
//                entries per shard (one ballot per shard per 32 entries);
//                counts are stored shard-major: [shard][warp]
//   2. scan    — ONE exclusive prefix sum over that flattened array is the
//                output offset of every (shard, warp) run (single CTA)
//   3. scatter — each warp re-reads its slice and writes every entry to
//                base[shard] + its rank among the warp's entries of that
//                shard; lane s keeps the running base of shard s (s < 64)
// Stable (input order within a shard is kept), streaming: 24 B read twice,
// 24 B written once per entry.
//
// Peer delivery (route_to_peers): the same count/scan, but the scatter writes
// each entry straight into its OWNER's receive arena — region [my_shard] of
// the owner's arena, over NVLink when the owner is another GPU (peer / IPC
// pointers) — and the scan publishes the bucket sizes into the owners' count
// arrays.  Route and all-to-all are one pass; no local bucket buffer, no NCCL.
#include "common.cuh"
#include "kernels.h"

namespace hetm_b200 {

constexpr int kRouteThreads = 256;
constexpr int kRouteWarps = kRouteThreads / 32;
constexpr int kMaxShards = 64;
constexpr int kScanThreads = 1024;
constexpr int kRouteUnroll = 4;  // 32-entry groups a warp loads before ranking them

__device__ __forceinline__ uint32_t owner_of(uint64_t addr, uint64_t shard_words, uint32_t n_shards) {
    uint64_t s = addr / shard_words;
    return (uint32_t)(s < n_shards ? s : n_shards - 1);
}

__device__ __forceinline__ void warp_slice(uint64_t n, uint64_t n_warps, uint64_t w, uint64_t& lo, uint64_t& hi) {
    lo = n * w / n_warps;
    hi = n * (w + 1) / n_warps;
}

__global__ void __launch_bounds__(kRouteThreads) route_count_kernel(const hetm_log_entry* __restrict__ in, uint64_t n,
                                                                    uint32_t nsh, uint64_t shard_words,
                                                                    unsigned long long* __restrict__ counts) {
    const uint64_t n_warps = (uint64_t)gridDim.x * kRouteWarps;
    const uint64_t w = (uint64_t)blockIdx.x * kRouteWarps + (threadIdx.x >> 5);
    const unsigned lane = lane_id();
    uint64_t lo, hi;
    warp_slice(n, n_warps, w, lo, hi);
    unsigned long long c0 = 0, c1 = 0;  // lane L counts shard L and shard L+32
    for (uint64_t i0 = lo; i0 < hi; i0 += 32 * kRouteUnroll) {
        uint32_t sv[kRouteUnroll];
#pragma unroll
        for (int u = 0; u < kRouteUnroll; ++u) {  // kRouteUnroll independent loads in flight per lane
            const uint64_t i = i0 + 32 * u + lane;
            sv[u] = i < hi ? owner_of(__ldg(&in[i].addr), shard_words, nsh) : 0xffffffffu;
        }
#pragma unroll
        for (int u = 0; u < kRouteUnroll; ++u) {
            for (uint32_t sh = 0; sh < nsh; ++sh) {
                const unsigned m = __ballot_sync(0xffffffffu, sv[u] == sh);
                if (lane == (sh & 31)) {
                    if (sh < 32) c0 += __popc(m);
                    else c1 += __popc(m);
                }
            }
        }
    }
    if (lane < nsh) counts[(uint64_t)lane * n_warps + w] = c0;
    if (lane + 32 < nsh) counts[(uint64_t)(lane + 32) * n_warps + w] = c1;
}

// Exclusive prefix sum of m values (one CTA): offsets[k] = sum_{j<k} counts[j];
// totals[s] = sum of shard s's segment [s*n_warps, (s+1)*n_warps).
__global__ void __launch_bounds__(kScanThreads) route_scan_kernel(const unsigned long long* __restrict__ counts,
                                                                  uint64_t n_warps, uint32_t nsh,
                                                                  unsigned long long* __restrict__ offsets,
                                                                  unsigned long long* __restrict__ totals) {
    __shared__ unsigned long long part[kScanThreads];
    const uint64_t m = n_warps * nsh;
    const uint64_t lo = m * threadIdx.x / kScanThreads, hi = m * (threadIdx.x + 1) / kScanThreads;
    unsigned long long sum = 0;
    for (uint64_t k = lo; k < hi; ++k) sum += counts[k];
    part[threadIdx.x] = sum;
    __syncthreads();
    for (int d = 1; d < kScanThreads; d <<= 1) {  // Hillis-Steele inclusive scan of the partial sums
        const unsigned long long x = threadIdx.x >= (unsigned)d ? part[threadIdx.x - d] : 0ull;
        __syncthreads();
        part[threadIdx.x] += x;
        __syncthreads();
    }
    unsigned long long run = part[threadIdx.x] - sum;
    for (uint64_t k = lo; k < hi; ++k) {
        offsets[k] = run;
        run += counts[k];
    }
    __syncthreads();
    for (uint32_t s = threadIdx.x; s < nsh; s += kScanThreads) {
        const unsigned long long start = offsets[(uint64_t)s * n_warps];
        const unsigned long long end =
            s + 1 < nsh ? offsets[(uint64_t)(s + 1) * n_warps] : offsets[m - 1] + counts[m - 1];
        totals[s] = end - start;
    }
}

// Peer variant of the scan epilogue: bucket sizes go to owner s's counts[my]
// and every offset becomes relative to its shard's bucket start.
__global__ void route_peer_publish_kernel(unsigned long long* offsets, const unsigned long long* totals,
                                          uint64_t n_warps, uint32_t nsh, uint32_t my,
                                          unsigned long long* const* peer_counts) {
    const uint32_t s = blockIdx.x;
    const unsigned long long start = offsets[(uint64_t)s * n_warps];
    __syncthreads();
    for (uint64_t w = threadIdx.x; w < n_warps; w += blockDim.x) offsets[(uint64_t)s * n_warps + w] -= start;
    if (threadIdx.x == 0) {
        peer_counts[s][my] = totals[s];
        __threadfence_system();  // the owner reads it after the round barrier
    }
}

__global__ void __launch_bounds__(kRouteThreads) route_scatter_kernel(const hetm_log_entry* __restrict__ in, uint64_t n,
                                                                      uint32_t nsh, uint64_t shard_words,
                                                                      const unsigned long long* __restrict__ offsets,
                                                                      hetm_log_entry* __restrict__ out) {
    const uint64_t n_warps = (uint64_t)gridDim.x * kRouteWarps;
    const uint64_t w = (uint64_t)blockIdx.x * kRouteWarps + (threadIdx.x >> 5);
    const unsigned lane = lane_id();
    uint64_t lo, hi;
    warp_slice(n, n_warps, w, lo, hi);
    unsigned long long b0 = lane < nsh ? offsets[(uint64_t)lane * n_warps + w] : 0;
    unsigned long long b1 = lane + 32 < nsh ? offsets[(uint64_t)(lane + 32) * n_warps + w] : 0;
    const unsigned lt = (1u << lane) - 1u;
    for (uint64_t i0 = lo; i0 < hi; i0 += 32 * kRouteUnroll) {
        hetm_log_entry ev[kRouteUnroll];
        uint32_t sv[kRouteUnroll];
#pragma unroll
        for (int u = 0; u < kRouteUnroll; ++u) {
            const uint64_t i = i0 + 32 * u + lane;
            sv[u] = 0xffffffffu;
            if (i < hi) {
                ev[u] = in[i];
                sv[u] = owner_of(ev[u].addr, shard_words, nsh);
            }
        }
#pragma unroll
        for (int u = 0; u < kRouteUnroll; ++u) {
            const uint32_t s = sv[u];
            unsigned rank = 0;
            const unsigned long long my0 = __shfl_sync(0xffffffffu, b0, s & 31);
            const unsigned long long my1 = __shfl_sync(0xffffffffu, b1, s & 31);
            for (uint32_t sh = 0; sh < nsh; ++sh) {
                const unsigned m = __ballot_sync(0xffffffffu, s == sh);
                if (s == sh) rank = __popc(m & lt);
                if (lane == (sh & 31)) {
                    if (sh < 32) b0 += __popc(m);
                    else b1 += __popc(m);
                }
            }
            if (s != 0xffffffffu) out[(s < 32 ? my0 : my1) + rank] = ev[u];
        }
    }
}

// Up to 8 CTAs per SM; small logs get fewer warps (>= 512 entries per warp) so
// the single-CTA scan over [shard][warp] stays short.
// Scatter into the owners' receive arenas: entry of shard s -> peer_out[s][my*cap + bucket offset].
__global__ void __launch_bounds__(kRouteThreads) route_peer_scatter_kernel(
    const hetm_log_entry* __restrict__ in, uint64_t n, uint32_t nsh, uint64_t shard_words,
    const unsigned long long* __restrict__ offsets, hetm_log_entry* const* peer_out, uint64_t region) {
    const uint64_t n_warps = (uint64_t)gridDim.x * kRouteWarps;
    const uint64_t w = (uint64_t)blockIdx.x * kRouteWarps + (threadIdx.x >> 5);
    const unsigned lane = lane_id();
    uint64_t lo, hi;
    warp_slice(n, n_warps, w, lo, hi);
    unsigned long long b0 = lane < nsh ? offsets[(uint64_t)lane * n_warps + w] : 0;
    unsigned long long b1 = lane + 32 < nsh ? offsets[(uint64_t)(lane + 32) * n_warps + w] : 0;
    hetm_log_entry* d0 = lane < nsh ? peer_out[lane] + region : nullptr;
    hetm_log_entry* d1 = lane + 32 < nsh ? peer_out[lane + 32] + region : nullptr;
    const unsigned lt = (1u << lane) - 1u;
    for (uint64_t i0 = lo; i0 < hi; i0 += 32 * kRouteUnroll) {
        hetm_log_entry ev[kRouteUnroll];
        uint32_t sv[kRouteUnroll];
#pragma unroll
        for (int u = 0; u < kRouteUnroll; ++u) {
            const uint64_t i = i0 + 32 * u + lane;
            sv[u] = 0xffffffffu;
            if (i < hi) {
                ev[u] = in[i];
                sv[u] = owner_of(ev[u].addr, shard_words, nsh);
            }
        }
#pragma unroll
        for (int u = 0; u < kRouteUnroll; ++u) {
            const uint32_t s = sv[u];
            unsigned rank = 0;
            const unsigned long long my0 = __shfl_sync(0xffffffffu, b0, s & 31);
            const unsigned long long my1 = __shfl_sync(0xffffffffu, b1, s & 31);
            hetm_log_entry* const p0 = reinterpret_cast<hetm_log_entry*>(
                __shfl_sync(0xffffffffu, reinterpret_cast<unsigned long long>(d0), s & 31));
            hetm_log_entry* const p1 = reinterpret_cast<hetm_log_entry*>(
                __shfl_sync(0xffffffffu, reinterpret_cast<unsigned long long>(d1), s & 31));
            for (uint32_t sh = 0; sh < nsh; ++sh) {
                const unsigned m = __ballot_sync(0xffffffffu, s == sh);
                if (s == sh) rank = __popc(m & lt);
                if (lane == (sh & 31)) {
                    if (sh < 32) b0 += __popc(m);
                    else b1 += __popc(m);
                }
            }
            if (s != 0xffffffffu) (s < 32 ? p0 + my0 : p1 + my1)[rank] = ev[u];
        }
    }
    // Peer stores over NVLink: make them visible system-wide before this kernel
    // completes, so the round barrier that follows on the stream (an NCCL
    // all-reduce, or a host barrier after a stream sync) orders them before
    // the owner's apply.
    __threadfence_system();
}

static unsigned route_grid(uint64_t n, const LaunchGeom& g) {
    const uint64_t want = (n + kRouteThreads * 16 - 1) / (kRouteThreads * 16);
    const uint64_t cap = (uint64_t)g.sm_count * 2u;  // each warp streams a long slice, 4 loads in flight
    return (unsigned)(want < 1 ? 1 : (want > cap ? cap : want));
}

size_t route_log_scratch_bytes(uint64_t n, uint32_t n_shards, const LaunchGeom& g) {
    return 2ull * route_grid(n, g) * kRouteWarps * n_shards * sizeof(unsigned long long);
}

cudaError_t launch_route_log(const hetm_log_entry* d_in, uint64_t n, uint32_t nsh, uint64_t shard_words,
                             hetm_log_entry* d_out, unsigned long long* d_counts, void* d_scratch, size_t scratch_bytes,
                             const LaunchGeom& g, cudaStream_t s) {
    if (nsh == 0 || nsh > kMaxShards || shard_words == 0) return cudaErrorInvalidValue;
    if (scratch_bytes < route_log_scratch_bytes(n, nsh, g)) return cudaErrorInvalidValue;
    const unsigned grid = route_grid(n, g);
    const uint64_t n_warps = (uint64_t)grid * kRouteWarps;
    auto* counts = static_cast<unsigned long long*>(d_scratch);
    auto* offsets = counts + n_warps * nsh;
    route_count_kernel<<<grid, kRouteThreads, 0, s>>>(d_in, n, nsh, shard_words, counts);
    route_scan_kernel<<<1, kScanThreads, 0, s>>>(counts, n_warps, nsh, offsets, d_counts);
    route_scatter_kernel<<<grid, kRouteThreads, 0, s>>>(d_in, n, nsh, shard_words, offsets, d_out);
    return cudaGetLastError();
}

cudaError_t launch_route_to_peers(const hetm_log_entry* d_in, uint64_t n, uint32_t nsh, uint64_t shard_words,
                                  uint32_t my, uint64_t cap, hetm_log_entry* const* d_peer_out,
                                  unsigned long long* const* d_peer_counts, unsigned long long* d_totals,
                                  void* d_scratch, size_t scratch_bytes, const LaunchGeom& g, cudaStream_t s) {
    if (nsh == 0 || nsh > kMaxShards || shard_words == 0 || my >= nsh || n > cap) return cudaErrorInvalidValue;
    if (scratch_bytes < route_log_scratch_bytes(n, nsh, g)) return cudaErrorInvalidValue;
    const unsigned grid = route_grid(n, g);
    const uint64_t n_warps = (uint64_t)grid * kRouteWarps;
    auto* counts = static_cast<unsigned long long*>(d_scratch);
    auto* offsets = counts + n_warps * nsh;
    route_count_kernel<<<grid, kRouteThreads, 0, s>>>(d_in, n, nsh, shard_words, counts);
    route_scan_kernel<<<1, kScanThreads, 0, s>>>(counts, n_warps, nsh, offsets, d_totals);
    route_peer_publish_kernel<<<nsh, 256, 0, s>>>(offsets, d_totals, n_warps, nsh, my, d_peer_counts);
    route_peer_scatter_kernel<<<grid, kRouteThreads, 0, s>>>(d_in, n, nsh, shard_words, offsets, d_peer_out,
                                                             (uint64_t)my * cap);
    return cudaGetLastError();
}

}  // namespace hetm_b200
