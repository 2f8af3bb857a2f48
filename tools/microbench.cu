// microbench.cu — B200 primitive costs that bound the HeTM device kernels.
// Not product code: measures random-access/atomic throughput so the kernel
// designs rest on numbers taken on this hardware.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o build/microbench tools/microbench.cu
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)

__device__ __forceinline__ uint64_t mix(uint64_t x) {
    x ^= x >> 33; x *= 0xff51afd7ed558ccdULL; x ^= x >> 33; x *= 0xc4ceb9fe1a85ec53ULL; x ^= x >> 33; return x;
}
__device__ __forceinline__ uint64_t ld_rlx(const uint64_t* p) {
    uint64_t v; asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory"); return v;
}

// mode 0: weak load, 1: relaxed.gpu load, 2: RED.MAX, 3: CAS (returns), 4: store, 5: load+store same addr
template <int MODE, int MLP>
__global__ void rand_access(uint64_t* a, uint64_t mask, uint64_t n_ops, uint64_t seed, unsigned long long* sink) {
    uint64_t tid = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    uint64_t acc = 0;
    for (uint64_t i = tid * MLP; i < n_ops; i += stride * MLP) {
        uint64_t idx[MLP];
#pragma unroll
        for (int k = 0; k < MLP; ++k) idx[k] = mix(seed + i + k) & mask;
        if (MODE == 0) {
            uint64_t v[MLP];
#pragma unroll
            for (int k = 0; k < MLP; ++k) v[k] = a[idx[k]];
#pragma unroll
            for (int k = 0; k < MLP; ++k) acc += v[k];
        } else if (MODE == 1) {
            uint64_t v[MLP];
#pragma unroll
            for (int k = 0; k < MLP; ++k) v[k] = ld_rlx(a + idx[k]);
#pragma unroll
            for (int k = 0; k < MLP; ++k) acc += v[k];
        } else if (MODE == 2) {
#pragma unroll
            for (int k = 0; k < MLP; ++k) atomicMax((unsigned long long*)a + idx[k], (unsigned long long)i);
        } else if (MODE == 3) {
            unsigned long long v[MLP];
#pragma unroll
            for (int k = 0; k < MLP; ++k) v[k] = atomicCAS((unsigned long long*)a + idx[k], 0ull, 1ull);
#pragma unroll
            for (int k = 0; k < MLP; ++k) acc += v[k];
        } else if (MODE == 4) {
#pragma unroll
            for (int k = 0; k < MLP; ++k) a[idx[k]] = i;
        } else if (MODE == 5) {
            uint64_t v[MLP];
#pragma unroll
            for (int k = 0; k < MLP; ++k) v[k] = ld_rlx(a + idx[k]);
#pragma unroll
            for (int k = 0; k < MLP; ++k) a[idx[k]] = v[k] + 1;
        }
    }
    if (acc == 0x1234567) atomicAdd(sink, 1ull);
}

// same-address ticket: one atomicAdd per warp per iteration
__global__ void ticket(unsigned long long* ctr, int iters) {
    for (int it = 0; it < iters; ++it) {
        unsigned long long b = 0;
        if ((threadIdx.x & 31) == 0) b = atomicAdd(ctr, 32ull);
        b = __shfl_sync(0xffffffffu, b, 0);
        if (b == 0xffffffffffffull) ctr[1] = b;
    }
}

// store; fence; store (release pattern) per iteration, random addresses
__global__ void fence_store(uint64_t* a, uint64_t mask, int iters, int use_fence) {
    uint64_t tid = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    for (int it = 0; it < iters; ++it) {
        uint64_t i1 = mix(tid * 1315423911ull + it) & mask, i2 = mix(tid * 2654435761ull + it + 7) & mask;
        a[i1] = it;
        if (use_fence) asm volatile("fence.acq_rel.gpu;" ::: "memory");
        asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(a + i2), "l"((uint64_t)it) : "memory");
    }
}

// dependent chain: pointer chase latency (1 thread per warp, many warps)
__global__ void chase(const uint64_t* a, uint64_t mask, int steps, unsigned long long* sink) {
    uint64_t p = mix(blockIdx.x * 977 + threadIdx.x) & mask;
    for (int s = 0; s < steps; ++s) p = (ld_rlx(a + p) + s) & mask;
    if (p == 0x12345) atomicAdd(sink, 1ull);
}

template <class F>
float timeit(F f, int reps = 5) {
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0); cudaEventCreate(&e1);
    f();
    cudaDeviceSynchronize();
    float best = 1e30f;
    for (int r = 0; r < reps; ++r) {
        cudaEventRecord(e0);
        f();
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        if (ms < best) best = ms;
    }
    return best;
}

int main() {
    int sms = 0; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const uint64_t W = 1ull << 27;  // 1 GiB of words
    uint64_t* a; CK(cudaMalloc(&a, W * 8)); CK(cudaMemset(a, 0, W * 8));
    unsigned long long* sink; CK(cudaMalloc(&sink, 64)); CK(cudaMemset(sink, 0, 64));
    // pointer-chase init: a[i] = random
    rand_access<4, 1><<<sms * 8, 256>>>(a, W - 1, W, 99, sink);
    CK(cudaDeviceSynchronize());
    const uint64_t N = 1ull << 24;  // ops per launch
    for (size_t gran : {(size_t)32, (size_t)64, (size_t)128, (size_t)0}) {
        cudaError_t e = cudaDeviceSetLimit(cudaLimitMaxL2FetchGranularity, gran);
        size_t got = 999;
        cudaDeviceGetLimit(&got, cudaLimitMaxL2FetchGranularity);
        float ms = timeit([&] { rand_access<1, 4><<<sms * 8, 256>>>(a, W - 1, N, 777, sink); });
        float ms2 = timeit([&] { rand_access<2, 4><<<sms * 8, 256>>>(a, W - 1, N, 778, sink); });
        printf("L2 fetch granularity set %zu (%s) -> reads %zu: random load %7.2f G/s, RED.MAX %7.2f G/s\n", gran,
               cudaGetErrorString(e), got, N / (ms * 1e6), N / (ms2 * 1e6));
    }
    if (getenv("MICRO_ONLY_GRAN")) return 0;
    const char* names[] = {"weak load", "relaxed.gpu load", "RED.MAX", "CAS", "store", "load+store"};
    for (uint64_t region : {W, W >> 3, W >> 6}) {  // 1 GiB, 128 MiB, 16 MiB
        for (int mode = 0; mode < 6; ++mode) {
            for (int occ : {4, 8}) {
                float ms;
                auto run = [&](auto kern) { ms = timeit([&] { kern<<<sms * occ, 256>>>(a, region - 1, N, 12345, sink); }); };
                switch (mode) {
                    case 0: run(rand_access<0, 4>); break;
                    case 1: run(rand_access<1, 4>); break;
                    case 2: run(rand_access<2, 4>); break;
                    case 3: run(rand_access<3, 4>); break;
                    case 4: run(rand_access<4, 4>); break;
                    case 5: run(rand_access<5, 4>); break;
                }
                printf("region %5llu MiB  %-18s blocks/SM %d : %8.3f ms  %7.2f G ops/s\n",
                       (unsigned long long)(region * 8 >> 20), names[mode], occ, ms, N / (ms * 1e6));
            }
        }
    }
    unsigned long long* ctr; CK(cudaMalloc(&ctr, 64)); CK(cudaMemset(ctr, 0, 64));
    for (int occ : {1, 4, 8}) {
        int iters = 64;
        float ms = timeit([&] { ticket<<<sms * occ, 256>>>(ctr, iters); });
        double n = (double)sms * occ * 8 * iters;
        printf("same-address warp ticket, %d blocks/SM: %.3f ms, %.1f M atomics/s (%.1f ns each)\n", occ, ms,
               n / (ms * 1e3), ms * 1e6 / n);
    }
    for (int f : {0, 1}) {
        int iters = 32;
        float ms = timeit([&] { fence_store<<<sms * 4, 256>>>(a, W - 1, iters, f); });
        printf("store;%sstore x%d per thread (%d thr): %.3f ms -> %.1f ns per iteration per thread-wave\n",
               f ? " fence.acq_rel;" : " ", iters, sms * 4 * 256, ms, ms * 1e6 / iters);
    }
    for (int warps : {1, 8, 32}) {
        int steps = 256;
        float ms = timeit([&] { chase<<<sms * warps, 1>>>(a, W - 1, steps, sink); }, 3);
        printf("pointer chase 1 GiB, %d chains/SM: %.3f ms -> %.0f ns per dependent load\n", warps, ms,
               ms * 1e6 / steps);
    }
    for (int warps : {1, 32}) {
        int steps = 256;
        float ms = timeit([&] { chase<<<sms * warps, 1>>>(a, (1ull << 21) - 1, steps, sink); }, 3);
        printf("pointer chase 16 MiB (L2), %d chains/SM: %.3f ms -> %.0f ns per dependent load\n", warps, ms,
               ms * 1e6 / steps);
    }
    return 0;
}
