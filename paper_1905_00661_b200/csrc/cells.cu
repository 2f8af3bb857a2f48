// cells.cu — conversions between the 32-B word-cell layout of devReplica
// (common.cuh) and plain 64-bit word arrays (devShadow, raw-op staging).
// Used at the edges only: raw ops, the shadow refresh of
// mergeCommit and the rollback of mergeAbortDevice.
#include <cstdlib>

#include <cub/device/device_radix_sort.cuh>

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

// mergeCommit delta: out[i] = {word, devReplica value} for every write-set
// log slot (duplicates carry the same final value; empty slots -> ~0 word),
// and the same value into devShadow (the incremental shadow refresh).
__global__ void wlog_gather_kernel(DeltaBuf out, uint64_t* __restrict__ shadow,
                                   const Cell* __restrict__ cells, const uint32_t* __restrict__ wlog, uint64_t n,
                                   uint64_t size_words) {
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t loc = wlog[i];
        if (loc < size_words && (i == 0 || wlog[i - 1] != loc)) {  // one record per word (the log is sorted)
            const uint64_t val = cells[loc].value;
            out.loc[i] = (uint32_t)loc;
            out.val[i] = val;
            if (shadow) shadow[loc] = val;
        } else {
            out.loc[i] = ~0u;
            out.val[i] = 0;
        }
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

cudaError_t launch_wlog_gather(DeltaBuf out, uint64_t* shadow, const Cell* cells, const uint32_t* wlog, uint64_t n,
                               uint64_t size_words, const LaunchGeom& g, cudaStream_t s) {
    if (n == 0) return cudaSuccess;
    wlog_gather_kernel<<<grid_words(n, g), 256, 0, s>>>(out, shadow, cells, wlog, n, size_words);
    return cudaGetLastError();
}

cudaError_t launch_delta_to_shadow(uint64_t* shadow, DeltaBuf d, uint64_t n, const LaunchGeom& g, cudaStream_t s) {
    if (n == 0) return cudaSuccess;
    delta_to_shadow_kernel<<<grid_words(n, g), 256, 0, s>>>(shadow, d, n);
    return cudaGetLastError();
}

// Sort the write-set log by word (CUB onesweep radix sort over the bits a
// local word index needs): the delta then reaches the host in address order,
// so each host worker scatters into one contiguous range of the replica.
// Empty slots (~0u) have all low bits set and sort last (a tie with word
// 2^bits-1 is harmless: the gather skips empty slots wherever they land).
static int sort_bits(uint64_t size_words) {
    int b = 1;
    while (b < 32 && (1ull << b) < size_words) ++b;
    return b;
}

size_t wlog_sort_temp_bytes(uint64_t n, uint64_t size_words) {
    size_t bytes = 0;
    cub::DeviceRadixSort::SortKeys(nullptr, bytes, (const uint32_t*)nullptr, (uint32_t*)nullptr, (int64_t)n, 0,
                                   sort_bits(size_words));
    return bytes;
}

cudaError_t launch_wlog_sort(const uint32_t* in, uint32_t* out, uint64_t n, uint64_t size_words, void* temp,
                             size_t temp_bytes, cudaStream_t s) {
    if (n == 0) return cudaSuccess;
    return cub::DeviceRadixSort::SortKeys(temp, temp_bytes, in, out, (int64_t)n, 0, sort_bits(size_words), s);
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
