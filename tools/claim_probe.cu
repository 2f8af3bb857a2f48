// claim_probe.cu — feasibility probe (not product code): a batch-synchronous
// "priority claim" schedule for bank transfers vs the product's PR-STM
// phases.  Per window of W txs: C kernel = each tx claims its 4 words with a
// fire-and-forget atomicMax(meta, epoch|~prio); E kernel = each tx re-reads
// its 4 {value, meta} cells and commits lock-free iff it holds all 4 claims
// (winners of one wave are pairwise disjoint).  E(k) is fused with C(k+1).
// Losers are counted, not retried (timing of the first wave only).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o build/claim_probe tools/claim_probe.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

struct alignas(16) Cell { unsigned long long value, meta; };
struct Tx { uint32_t a[4]; uint64_t amount; };

__device__ __forceinline__ uint64_t mix(uint64_t x) {
    x ^= x >> 33; x *= 0xff51afd7ed558ccdULL; x ^= x >> 33; x *= 0xc4ceb9fe1a85ec53ULL; x ^= x >> 33; return x;
}
__global__ void gen(Tx* t, uint64_t n, uint64_t W) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
        for (int k = 0; k < 4; ++k) t[i].a[k] = (uint32_t)(mix(i * 4 + k + 1) % W);
        t[i].amount = 1 + i % 100;
    }
}
__device__ __forceinline__ unsigned long long key_of(uint32_t epoch, uint64_t i) {
    return (1ull << 63) | ((unsigned long long)epoch << 32) | (0xffffffffull - (i & 0xffffffffull));
}
// one launch: execute window `ex` (epoch e) and claim window `cl` (epoch e+1)
__global__ void stage(Cell* c, const Tx* t, uint64_t ex_lo, uint64_t ex_n, uint64_t cl_lo, uint64_t cl_n, uint32_t e,
                      unsigned long long* wins, unsigned long long* ticket) {
    const uint64_t n = ex_n + cl_n;
    unsigned long long won = 0;
    for (uint64_t j = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; j < n; j += (uint64_t)gridDim.x * blockDim.x) {
        if (j >= ex_n) {  // claim
            const uint64_t i = cl_lo + (j - ex_n);
            const unsigned long long k = key_of(e + 1, i);
            for (int q = 0; q < 4; ++q) atomicMax(&c[t[i].a[q]].meta, k);
        } else {  // execute
            const uint64_t i = ex_lo + j;
            const unsigned long long k = key_of(e, i);
            unsigned long long v[4], m[4];
            for (int q = 0; q < 4; ++q) {
                asm volatile("ld.relaxed.gpu.global.v2.u64 {%0,%1}, [%2];" : "=l"(v[q]), "=l"(m[q]) : "l"(&c[t[i].a[q]]) : "memory");
            }
            bool ok = true;
            for (int q = 0; q < 4; ++q) ok &= (m[q] == k);
            // warp-aggregated ticket over the winning lanes
            const unsigned am = __activemask();
            const unsigned wm = __ballot_sync(am, ok);
            unsigned long long base = 0;
            const unsigned lead = __ffs(am) - 1, lane = threadIdx.x & 31;
            if (lane == lead && wm) base = atomicAdd(ticket, (unsigned long long)__popc(wm));
            base = __shfl_sync(am, base, lead);
            if (ok) {
                const unsigned long long tk = base + __popc(wm & ((1u << lane) - 1u));
                const unsigned long long nm = (tk + 1) & 0x7fffffffull;
                c[t[i].a[0]] = Cell{v[0] - t[i].amount, nm};
                c[t[i].a[1]] = Cell{v[1] + t[i].amount, nm};
                c[t[i].a[2]].meta = nm;
                c[t[i].a[3]].meta = nm;
                ++won;
            }
        }
    }
    if (won) atomicAdd(wins, won);
}

int main() {
    const uint64_t W = 1ull << 27, N = 1ull << 20;
    Cell* c; Tx* t; unsigned long long *wins, *ticket;
    cudaMalloc(&c, W * sizeof(Cell)); cudaMemset(c, 0, W * sizeof(Cell));
    cudaMalloc(&t, N * sizeof(Tx)); cudaMalloc(&wins, 8); cudaMalloc(&ticket, 8);
    gen<<<1184, 256>>>(t, N, W / 2);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    for (uint64_t win : {1ull << 16, 1ull << 17, 1ull << 18, 1ull << 20}) {
        for (int bps : {1, 4}) {
            for (int rep = 0; rep < 3; ++rep) {
                cudaMemset(wins, 0, 8);
                uint32_t e = (uint32_t)(rep * 64 + 1);
                cudaEventRecord(a);
                uint64_t prev_lo = 0, prev_n = 0;
                for (uint64_t lo = 0; lo < N || prev_n; lo += win) {
                    const uint64_t n = lo < N ? (N - lo < win ? N - lo : win) : 0;
                    stage<<<148 * bps, 256>>>(c, t, prev_lo, prev_n, lo, n, e, wins, ticket);
                    prev_lo = lo; prev_n = n; ++e;
                }
                cudaEventRecord(b); cudaEventSynchronize(b);
                float ms; cudaEventElapsedTime(&ms, a, b);
                unsigned long long w; cudaMemcpy(&w, wins, 8, cudaMemcpyDeviceToHost);
                if (rep) printf("window 2^%d CTAs/SM %d: %.4f ms for %llu tx (first-wave winners %.2f%%) -> %.2f G tx/s\n",
                                __builtin_ctzll(win), bps, ms, (unsigned long long)N, 100.0 * w / N, N / ms / 1e6);
            }
        }
    }
    return 0;
}
