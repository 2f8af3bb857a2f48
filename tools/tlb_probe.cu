// tlb_probe.cu — random 16-B load / CAS throughput vs. footprint (TLB reach probe).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__device__ __forceinline__ uint64_t mix(uint64_t x) {
    x ^= x >> 33; x *= 0xff51afd7ed558ccdULL; x ^= x >> 33; x *= 0xc4ceb9fe1a85ec53ULL; x ^= x >> 33; return x;
}
template <int MODE>
__global__ void k(uint64_t* a, uint64_t cells_mask, uint64_t n, unsigned long long* sink) {
    uint64_t acc = 0;
    for (uint64_t i = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) * 4; i < n; i += (uint64_t)gridDim.x * blockDim.x * 4) {
        uint64_t idx[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) idx[q] = (mix(i + q) & cells_mask) * 4;  // 32-B cells
        if (MODE == 0) {
            uint64_t v[4];
#pragma unroll
            for (int q = 0; q < 4; ++q) asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v[q]) : "l"(a + idx[q]) : "memory");
#pragma unroll
            for (int q = 0; q < 4; ++q) acc += v[q];
        } else {
#pragma unroll
            for (int q = 0; q < 4; ++q) acc += atomicCAS((unsigned long long*)a + idx[q] + 1, 0ull, 0ull);
        }
    }
    if (acc == 12345) atomicAdd(sink, 1ull);
}
int main() {
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const uint64_t maxb = 32ull << 30;
    uint64_t* a; if (cudaMalloc(&a, maxb) != cudaSuccess) { printf("alloc fail\n"); return 1; }
    cudaMemset(a, 0, maxb);
    unsigned long long* sink; cudaMalloc(&sink, 8);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    const uint64_t n = 1ull << 24;
    for (uint64_t gib : {1ull, 2ull, 4ull, 8ull, 16ull, 32ull}) {
        uint64_t cells = (gib << 30) / 32;
        for (int mode = 0; mode < 2; ++mode) {
            float best = 1e9;
            for (int r = 0; r < 4; ++r) {
                cudaEventRecord(e0);
                if (mode == 0) k<0><<<sms * 8, 256>>>(a, cells - 1, n, sink);
                else k<1><<<sms * 8, 256>>>(a, cells - 1, n, sink);
                cudaEventRecord(e1); cudaEventSynchronize(e1);
                float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms;
            }
            printf("%3llu GiB footprint  %s: %7.2f G ops/s\n", (unsigned long long)gib, mode ? "CAS " : "load", n / (best * 1e6));
        }
    }
    return 0;
}
