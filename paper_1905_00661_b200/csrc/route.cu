// route.cu — shard router for address-range sharded validation.
//
// Shard s owns global words [s*shard_words, (s+1)*shard_words).  The router
// stable-partitions a log buffer by owner shard so the buckets can be sent
// all-to-all (NCCL over NVLink) and validated/applied locally by the owner.
// Three launches: per-CTA counts -> one-CTA scan -> in-order ballot scatter.
#include "common.cuh"
#include "kernels.h"

namespace hetm_b200 {

constexpr int kRouteThreads = 256;
constexpr int kRouteGrid = 592;  // 4 CTAs per SM on 148 SMs; each CTA owns one contiguous range
constexpr int kMaxShards = 64;

__device__ __forceinline__ uint32_t owner_of(uint64_t addr, uint64_t shard_words, uint32_t n_shards) {
    uint64_t s = addr / shard_words;
    return (uint32_t)(s < n_shards ? s : n_shards - 1);
}

__global__ void route_count_kernel(const hetm_log_entry* __restrict__ in, uint64_t n, uint32_t nsh,
                                   uint64_t shard_words, unsigned long long* counts) {
    __shared__ unsigned long long c[kMaxShards];
    for (uint32_t s = threadIdx.x; s < nsh; s += blockDim.x) c[s] = 0;
    __syncthreads();
    const uint64_t lo = n * blockIdx.x / gridDim.x, hi = n * (blockIdx.x + 1) / gridDim.x;
    for (uint64_t i = lo + threadIdx.x; i < hi; i += blockDim.x)
        atomicAdd(&c[owner_of(__ldg(&in[i].addr), shard_words, nsh)], 1ull);
    __syncthreads();
    for (uint32_t s = threadIdx.x; s < nsh; s += blockDim.x) counts[(uint64_t)blockIdx.x * nsh + s] = c[s];
}

// offsets[b*nsh+s] = sum_{s'<s} total[s'] + sum_{b'<b} counts[b'][s]
__global__ void route_scan_kernel(const unsigned long long* counts, uint32_t grid, uint32_t nsh,
                                  unsigned long long* offsets, unsigned long long* totals) {
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    unsigned long long run = 0;
    for (uint32_t s = 0; s < nsh; ++s) {
        unsigned long long start = run;
        for (uint32_t b = 0; b < grid; ++b) {
            offsets[(uint64_t)b * nsh + s] = run;
            run += counts[(uint64_t)b * nsh + s];
        }
        totals[s] = run - start;
    }
}

__global__ void __launch_bounds__(kRouteThreads) route_scatter_kernel(const hetm_log_entry* __restrict__ in, uint64_t n,
                                                                      uint32_t nsh, uint64_t shard_words,
                                                                      const unsigned long long* offsets,
                                                                      hetm_log_entry* __restrict__ out) {
    constexpr int kWarps = kRouteThreads / 32;
    __shared__ unsigned long long base[kMaxShards];
    __shared__ unsigned warp_cnt[kWarps][kMaxShards];
    __shared__ unsigned warp_pre[kWarps][kMaxShards];
    __shared__ unsigned tile_tot[kMaxShards];
    for (uint32_t s = threadIdx.x; s < nsh; s += blockDim.x) base[s] = offsets[(uint64_t)blockIdx.x * nsh + s];
    __syncthreads();
    const uint64_t lo = n * blockIdx.x / gridDim.x, hi = n * (blockIdx.x + 1) / gridDim.x;
    const unsigned warp = threadIdx.x >> 5, lane = lane_id();
    for (uint64_t t0 = lo; t0 < hi; t0 += blockDim.x) {
        const uint64_t i = t0 + threadIdx.x;
        const bool valid = i < hi;
        hetm_log_entry e{};
        uint32_t s = 0xffffffffu;
        if (valid) {
            e = in[i];
            s = owner_of(e.addr, shard_words, nsh);
        }
        unsigned my_rank = 0;
        for (uint32_t sh = 0; sh < nsh; ++sh) {
            unsigned m = __ballot_sync(0xffffffffu, s == sh);
            if (s == sh) my_rank = __popc(m & ((1u << lane) - 1u));
            if (lane == 0) warp_cnt[warp][sh] = __popc(m);
        }
        __syncthreads();
        for (uint32_t sh = threadIdx.x; sh < nsh; sh += blockDim.x) {
            unsigned run = 0;
            for (int w = 0; w < kWarps; ++w) {
                warp_pre[w][sh] = run;
                run += warp_cnt[w][sh];
            }
            tile_tot[sh] = run;
        }
        __syncthreads();
        if (valid) out[base[s] + warp_pre[warp][s] + my_rank] = e;
        __syncthreads();
        for (uint32_t sh = threadIdx.x; sh < nsh; sh += blockDim.x) base[sh] += tile_tot[sh];
        __syncthreads();
    }
}

size_t route_log_scratch_bytes(uint64_t, uint32_t n_shards) {
    return 2ull * kRouteGrid * n_shards * sizeof(unsigned long long);
}

cudaError_t launch_route_log(const hetm_log_entry* d_in, uint64_t n, uint32_t nsh, uint64_t shard_words,
                             hetm_log_entry* d_out, unsigned long long* d_counts, void* d_scratch, size_t scratch_bytes,
                             cudaStream_t s) {
    if (nsh == 0 || nsh > kMaxShards || shard_words == 0) return cudaErrorInvalidValue;
    if (scratch_bytes < route_log_scratch_bytes(n, nsh)) return cudaErrorInvalidValue;
    auto* counts = static_cast<unsigned long long*>(d_scratch);
    auto* offsets = counts + (size_t)kRouteGrid * nsh;
    route_count_kernel<<<kRouteGrid, kRouteThreads, 0, s>>>(d_in, n, nsh, shard_words, counts);
    route_scan_kernel<<<1, 32, 0, s>>>(counts, kRouteGrid, nsh, offsets, d_counts);
    route_scatter_kernel<<<kRouteGrid, kRouteThreads, 0, s>>>(d_in, n, nsh, shard_words, offsets, d_out);
    return cudaGetLastError();
}

}  // namespace hetm_b200
