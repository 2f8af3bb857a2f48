// cas_probe.cu — what does a lock CAS on a just-filled random line cost on B200?
// (not product code).  Each thread: 4 random 16-B cell loads, then per mode:
//   0 floor: 2 stores                   1: 2 CAS that succeed, then 2 stores
//   2: 2 CAS that fail (no write), then 2 stores
//   3: 2 atomicOr (RMW, returns), then 2 stores      4: 2 RED.OR (no return), then 2 stores
//   5: 2 loads again (L2 hit round trip), then 2 stores
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o build/cas_probe tools/cas_probe.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

struct alignas(16) Cell { unsigned long long value, meta; };
__device__ __forceinline__ uint64_t mix(uint64_t x) {
    x ^= x >> 33; x *= 0xff51afd7ed558ccdULL; x ^= x >> 33; x *= 0xc4ceb9fe1a85ec53ULL; x ^= x >> 33; return x;
}
template <int MODE>
__global__ void k(Cell* c, uint64_t W, uint64_t n, uint64_t seed, unsigned long long* sink) {
    unsigned long long acc = 0;
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
        uint64_t a[4];
        unsigned long long v[4], m[4];
        for (int q = 0; q < 4; ++q) a[q] = mix(seed + 4 * i + q) % W;
        for (int q = 0; q < 4; ++q)
            asm volatile("ld.relaxed.gpu.global.v2.u64 {%0,%1}, [%2];" : "=l"(v[q]), "=l"(m[q]) : "l"(&c[a[q]]) : "memory");
        if (MODE == 1 || MODE == 2) {
            unsigned long long r[2];
            for (int q = 0; q < 2; ++q)
                r[q] = atomicCAS(&c[a[q]].meta, MODE == 1 ? m[q] : ~m[q], m[q] | (1ull << 63));
            acc += r[0] ^ r[1];
        } else if (MODE == 3) {
            unsigned long long r[2];
            for (int q = 0; q < 2; ++q) r[q] = atomicOr(&c[a[q]].meta, 1ull << 62);
            acc += r[0] ^ r[1];
        } else if (MODE == 4) {
            for (int q = 0; q < 2; ++q) atomicOr(&c[a[q]].meta, 1ull << 61);
        } else if (MODE == 5) {
            unsigned long long r[2];
            for (int q = 0; q < 2; ++q)
                asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(r[q]) : "l"(&c[a[q]].meta) : "memory");
            acc += r[0] ^ r[1];
        }
        for (int q = 0; q < 2; ++q) {
            c[a[q]].value = v[q] + 1;
            c[a[q]].meta = m[q] & 0xffffffffull;
        }
        acc += v[2] + v[3];
    }
    if (acc == 42) *sink = acc;
}

int main() {
    const uint64_t W = 1ull << 27, N = 1ull << 20;
    Cell* c; unsigned long long* sink;
    cudaMalloc(&c, W * sizeof(Cell)); cudaMemset(c, 0, W * sizeof(Cell)); cudaMalloc(&sink, 8);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    const char* names[] = {"floor: load4 + store2", "load4 + CAS2 (succeed) + store2", "load4 + CAS2 (fail) + store2",
                           "load4 + atomicOr2 (returning) + store2", "load4 + RED.OR2 + store2",
                           "load4 + load2 again + store2"};
    for (int bps : {1, 4}) {
        for (int mode = 0; mode < 6; ++mode) {
            float best = 1e9;
            for (int rep = 0; rep < 4; ++rep) {
                cudaEventRecord(a);
                switch (mode) {
                    case 0: k<0><<<148 * bps, 256>>>(c, W, N, rep * N * 8, sink); break;
                    case 1: k<1><<<148 * bps, 256>>>(c, W, N, rep * N * 8, sink); break;
                    case 2: k<2><<<148 * bps, 256>>>(c, W, N, rep * N * 8, sink); break;
                    case 3: k<3><<<148 * bps, 256>>>(c, W, N, rep * N * 8, sink); break;
                    case 4: k<4><<<148 * bps, 256>>>(c, W, N, rep * N * 8, sink); break;
                    case 5: k<5><<<148 * bps, 256>>>(c, W, N, rep * N * 8, sink); break;
                }
                cudaEventRecord(b); cudaEventSynchronize(b);
                float ms; cudaEventElapsedTime(&ms, a, b);
                if (rep && ms < best) best = ms;
            }
            printf("CTAs/SM %d  %-42s %.4f ms  (%.2f G tx-shapes/s)\n", bps, names[mode], best, N / best / 1e6);
        }
    }
    return 0;
}
