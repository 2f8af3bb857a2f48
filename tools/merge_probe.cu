// merge_probe.cu — how to deliver a sparse device write set into the host
// replica (not product code; numbers decide the merge design in DESIGN.md).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -Xcompiler -fopenmp -o build/merge_probe tools/merge_probe.cu
// A: full 512 MiB D2H (the SPEC chunk copy when every chunk is dirty)
// B: GPU zero-copy scatter of n random 8-B words into mapped pinned host memory
// C: D2H of the compact {loc,value} delta (16 B/word) + host OpenMP scatter
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <chrono>
#include <vector>
#include <omp.h>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)

__device__ __forceinline__ uint64_t mix(uint64_t x) {
    x ^= x >> 33; x *= 0xff51afd7ed558ccdULL; x ^= x >> 33; x *= 0xc4ceb9fe1a85ec53ULL; x ^= x >> 33; return x;
}
struct Delta { uint64_t loc, value; };

__global__ void make_delta(Delta* d, uint64_t n, uint64_t mask) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
        d[i] = Delta{mix(i + 1) & mask, i};
}
__global__ void zc_scatter(uint64_t* host, const Delta* d, uint64_t n) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
        const Delta x = d[i];
        host[x.loc] = x.value;
    }
}

static double now() { return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count(); }

int main() {
    const uint64_t W = 1ull << 26;  // 512 MiB of words (the GPU half of a 1 GiB shard)
    uint64_t *h_rep = nullptr, *d_rep = nullptr;
    CK(cudaHostAlloc(&h_rep, W * 8, cudaHostAllocMapped | cudaHostAllocPortable));
    CK(cudaMalloc(&d_rep, W * 8));
    CK(cudaMemset(d_rep, 1, W * 8));
    for (uint64_t i = 0; i < W; ++i) h_rep[i] = 0;
    uint64_t* h_dev_ptr = nullptr;
    CK(cudaHostGetDevicePointer((void**)&h_dev_ptr, h_rep, 0));
    cudaEvent_t a, b;
    cudaEventCreate(&a); cudaEventCreate(&b);
    // A
    for (int r = 0; r < 3; ++r) {
        cudaEventRecord(a);
        CK(cudaMemcpyAsync(h_rep, d_rep, W * 8, cudaMemcpyDeviceToHost));
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms; cudaEventElapsedTime(&ms, a, b);
        printf("A full D2H 512 MiB: %.3f ms (%.1f GB/s)\n", ms, W * 8 / ms / 1e6);
    }
    printf("host threads: %d\n", omp_get_max_threads());
    for (uint64_t n : {1ull << 18, 1ull << 20, 1ull << 21, 1ull << 22}) {
        Delta* d_delta; Delta* h_delta;
        CK(cudaMalloc(&d_delta, n * sizeof(Delta)));
        CK(cudaHostAlloc(&h_delta, n * sizeof(Delta), cudaHostAllocPortable));
        make_delta<<<1184, 256>>>(d_delta, n, W - 1);
        CK(cudaDeviceSynchronize());
        for (int r = 0; r < 2; ++r) {
            for (int grid : {148, 592, 2368}) {
                cudaEventRecord(a);
                zc_scatter<<<grid, 256>>>(h_dev_ptr, d_delta, n);
                cudaEventRecord(b);
                CK(cudaEventSynchronize(b));
                float ms; cudaEventElapsedTime(&ms, a, b);
                printf("B zero-copy scatter n=%llu grid=%d: %.3f ms (%.1f M words/s)\n", (unsigned long long)n, grid, ms,
                       n / ms / 1e3);
            }
            // C: pipelined pieces
            const uint64_t piece = 1ull << 17;
            std::vector<cudaEvent_t> ev((n + piece - 1) / piece);
            for (auto& e : ev) cudaEventCreateWithFlags(&e, cudaEventDisableTiming);
            double t0 = now();
            for (size_t k = 0; k < ev.size(); ++k) {
                const uint64_t lo = k * piece, m = std::min(piece, n - lo);
                CK(cudaMemcpyAsync(h_delta + lo, d_delta + lo, m * sizeof(Delta), cudaMemcpyDeviceToHost));
                cudaEventRecord(ev[k]);
            }
            for (size_t k = 0; k < ev.size(); ++k) {
                cudaEventSynchronize(ev[k]);
                const uint64_t lo = k * piece, m = std::min(piece, n - lo);
#pragma omp parallel for schedule(static)
                for (int64_t i = 0; i < (int64_t)m; ++i) h_rep[h_delta[lo + i].loc] = h_delta[lo + i].value;
            }
            double t1 = now();
            printf("C delta D2H + host scatter n=%llu: %.3f ms (%.1f M words/s)\n", (unsigned long long)n,
                   (t1 - t0) * 1e3, n / (t1 - t0) / 1e6);
            for (auto& e : ev) cudaEventDestroy(e);
        }
        cudaFree(d_delta); cudaFreeHost(h_delta);
    }
    return 0;
}
