// tlb_probe2.cu — is the ~40 G/s random-access ceiling on a 2 GiB buffer set by
// address translation (TLB reach) rather than DRAM?  (not product code)
//
// Each thread runs `iters` iterations; per iteration 4 random 16-B loads of a
// 2 GiB cell array (+ optionally 2 dependent re-loads of the same cells, the
// bank kernel's P2/P4 shape).  Address choice:
//   rand   uniform over the whole buffer (1024 x 2 MiB pages)
//   local  uniform within a window of 16 pages (32 MiB) that all threads move
//          through together (iteration i uses pages [16*(i % 64), +16)): the
//          same DRAM randomness inside pages, few pages in flight
// Allocation: cudaMalloc, or cuMemCreate/cuMemMap with the largest granularity
// the driver reports (VMM).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o build/tlb_probe2 tools/tlb_probe2.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

struct alignas(16) Cell {
    unsigned long long value, meta;
};
__device__ __forceinline__ uint64_t mix(uint64_t x) {
    x ^= x >> 33;
    x *= 0xff51afd7ed558ccdULL;
    x ^= x >> 33;
    x *= 0xc4ceb9fe1a85ec53ULL;
    x ^= x >> 33;
    return x;
}

template <bool LOCAL, bool RELOAD>
__global__ void k(Cell* c, uint64_t W, int iters, uint64_t seed, unsigned long long* sink) {
    const uint64_t tid = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    constexpr uint64_t kPageCells = (2ull << 20) / sizeof(Cell);
    const uint64_t pages = W / kPageCells;
    unsigned long long acc = 0;
    for (int it = 0; it < iters; ++it) {
        uint64_t a[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const uint64_t h = mix(seed + (tid * iters + it) * 4 + q);
            if (LOCAL) {
                const uint64_t page = (16 * (uint64_t)(it % 64) + (h >> 40) % 16) % pages;
                a[q] = page * kPageCells + (h % kPageCells);
            } else {
                a[q] = h % W;
            }
        }
        unsigned long long v[4], m[4];
#pragma unroll
        for (int q = 0; q < 4; ++q)
            asm volatile("ld.relaxed.gpu.global.v2.u64 {%0,%1}, [%2];" : "=l"(v[q]), "=l"(m[q]) : "l"(&c[a[q]]) : "memory");
        if (RELOAD) {  // dependent on the first loads (the bank kernel's CAS / validation round trip)
            unsigned long long r[2];
#pragma unroll
            for (int q = 0; q < 2; ++q)
                asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];"
                             : "=l"(r[q])
                             : "l"(&c[a[q] ^ (m[q] & v[q] & 0x8000000000000000ull ? 1 : 0)].meta)
                             : "memory");
            acc += r[0] ^ r[1];
        }
        acc += v[0] + v[1] + v[2] + v[3] + m[0];
    }
    if (acc == 42) *sink = acc;
}

template <bool L, bool R>
float run(Cell* c, uint64_t W, int grid, int threads, int iters, unsigned long long* sink) {
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    k<L, R><<<grid, threads>>>(c, W, iters, 7, sink);  // warm-up
    cudaEventRecord(a);
    k<L, R><<<grid, threads>>>(c, W, iters, 11, sink);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    return ms;
}

void sweep(const char* alloc, Cell* c, uint64_t W, int sms, unsigned long long* sink) {
    const int iters = 64;
    for (int bps : {1, 4}) {
        const int grid = sms * bps, threads = 256;
        const double n = (double)grid * threads * iters;
        const float a = run<false, false>(c, W, grid, threads, iters, sink);
        const float b = run<true, false>(c, W, grid, threads, iters, sink);
        const float d = run<false, true>(c, W, grid, threads, iters, sink);
        const float e = run<true, true>(c, W, grid, threads, iters, sink);
        printf("%-28s CTAs/SM %d  rand load4 %6.2f G loads/s | local load4 %6.2f | rand load4+reload2 %6.2f G acc/s "
               "| local load4+reload2 %6.2f\n",
               alloc, bps, 4 * n / a / 1e6, 4 * n / b / 1e6, 6 * n / d / 1e6, 6 * n / e / 1e6);
    }
}

int main() {
    const uint64_t W = 1ull << 27;  // 2 GiB of 16-B cells
    const size_t bytes = W * sizeof(Cell);
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    unsigned long long* sink;
    cudaMalloc(&sink, 8);
    Cell* c = nullptr;
    cudaMalloc(&c, bytes);
    cudaMemset(c, 0, bytes);
    sweep("cudaMalloc", c, W, sms, sink);
    cudaFree(c);

    cuInit(0);
    CUdevice dev;
    cuDeviceGet(&dev, 0);
    CUmemAllocationProp prop = {};
    prop.type = CU_MEM_ALLOCATION_TYPE_PINNED;
    prop.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
    prop.location.id = 0;
    size_t gmin = 0, grec = 0;
    cuMemGetAllocationGranularity(&gmin, &prop, CU_MEM_ALLOC_GRANULARITY_MINIMUM);
    cuMemGetAllocationGranularity(&grec, &prop, CU_MEM_ALLOC_GRANULARITY_RECOMMENDED);
    printf("VMM granularity: minimum %zu B, recommended %zu B\n", gmin, grec);
    for (size_t chunk : {(size_t)bytes, (size_t)(512ull << 20), (size_t)(2ull << 20)}) {
        if (chunk % gmin) continue;
        CUdeviceptr va = 0;
        if (cuMemAddressReserve(&va, bytes, chunk > (1ull << 30) ? (1ull << 30) : chunk, 0, 0) != CUDA_SUCCESS) {
            printf("reserve failed\n");
            continue;
        }
        bool ok = true;
        CUmemGenericAllocationHandle hs[1024];
        const size_t nch = bytes / chunk;
        for (size_t q = 0; q < nch && ok; ++q) {
            ok = cuMemCreate(&hs[q], chunk, &prop, 0) == CUDA_SUCCESS &&
                 cuMemMap(va + q * chunk, chunk, 0, hs[q], 0) == CUDA_SUCCESS;
        }
        CUmemAccessDesc ad = {};
        ad.location = prop.location;
        ad.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
        ok = ok && cuMemSetAccess(va, bytes, &ad, 1) == CUDA_SUCCESS;
        if (ok) {
            cudaMemset((void*)va, 0, bytes);
            char name[64];
            snprintf(name, sizeof name, "VMM chunks of %zu MiB", chunk >> 20);
            sweep(name, (Cell*)va, W, sms, sink);
        } else {
            printf("VMM mapping with %zu MiB chunks failed\n", chunk >> 20);
        }
        cuMemUnmap(va, bytes);
        for (size_t q = 0; q < nch; ++q) cuMemRelease(hs[q]);
        cuMemAddressFree(va, bytes);
    }
    cudaError_t e = cudaDeviceSynchronize();
    printf("done: %s\n", cudaGetErrorString(e));
    return 0;
}
