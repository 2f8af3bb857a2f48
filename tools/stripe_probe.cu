// stripe_probe.cu — would an L2-resident lock-stripe table beat per-cell locks
// for the bank commit, and what does a single-access apply cost? (not product
// code).  W = 2^27 16-B cells (2 GiB, >> L2), 2^20 transactions of 4 random
// accounts (a0, a1 read-modify-written; a2, a3 read-only, values unused).
//
//   cell   : today's shape — P1 ld.v2 a0,a1 + ld meta a2,a3 (DRAM); P2 CAS
//            meta a0,a1; P4 reload meta a2,a3; P5 st.v2 a0,a1
//   stripe : P0 ld.acquire 4 stripe words (L2-resident table); P1 ld.v2 a0,a1;
//            P2 CAS stripes a0,a1; P4 reload stripes a2,a3; P5 st.v2 a0,a1,
//            fence, release stripes a0,a1
//   stripe-nofence : same without the acquire / fence (cost of ordering)
//   floor  : P1 ld.v2 a0,a1; P5 st.v2 a0,a1
// Apply (2^20 log entries of 24 B, uniform words):
//   amax   : returning atomicMax(meta, ts); if raised, store value (today)
//   blind  : one 16-B store {value, ts} per entry
//   table  : RED.MAX ts into an L2 table slot (kernel 1); load slot, blind
//            16-B store if own ts is the slot max (kernel 2)
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o build/stripe_probe tools/stripe_probe.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

struct alignas(16) Cell { unsigned long long value, meta; };
__device__ __forceinline__ uint64_t mix(uint64_t x) {
    x ^= x >> 33; x *= 0xff51afd7ed558ccdULL; x ^= x >> 33; x *= 0xc4ceb9fe1a85ec53ULL; x ^= x >> 33; return x;
}
__device__ __forceinline__ void ldv2(const Cell* p, unsigned long long& v, unsigned long long& m) {
    asm volatile("ld.relaxed.gpu.global.v2.u64 {%0,%1}, [%2];" : "=l"(v), "=l"(m) : "l"(p) : "memory");
}
__device__ __forceinline__ void stv2(Cell* p, unsigned long long v, unsigned long long m) {
    asm volatile("st.relaxed.gpu.global.v2.u64 [%0], {%1,%2};" ::"l"(p), "l"(v), "l"(m) : "memory");
}
__device__ __forceinline__ unsigned long long ld_rlx(const unsigned long long* p) {
    unsigned long long r;
    asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(r) : "l"(p) : "memory");
    return r;
}
__device__ __forceinline__ unsigned long long ld_acq(const unsigned long long* p) {
    unsigned long long r;
    asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(r) : "l"(p) : "memory");
    return r;
}

template <int MODE>  // 0 floor, 1 cell, 2 stripe, 3 stripe-nofence
__global__ void tx(Cell* c, unsigned long long* st, uint64_t W, uint32_t smask, uint32_t sshift, uint64_t n,
                   uint64_t seed, unsigned long long* sink) {
    unsigned long long acc = 0;
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
        uint64_t a[4];
        for (int q = 0; q < 4; ++q) a[q] = mix(seed + 4 * i + q) % W;
        unsigned long long v[2], m[4], s[4];
        if (MODE == 2 || MODE == 3) {
            for (int q = 0; q < 4; ++q) {
                const uint32_t si = (uint32_t)(mix(a[q] >> sshift) & smask);
                s[q] = MODE == 2 ? ld_acq(&st[si]) : ld_rlx(&st[si]);
            }
        }
        for (int q = 0; q < 2; ++q) ldv2(&c[a[q]], v[q], m[q]);
        if (MODE == 1)
            for (int q = 2; q < 4; ++q) m[q] = ld_rlx(&c[a[q]].meta);
        if (MODE == 1) {
            for (int q = 0; q < 2; ++q) acc += atomicCAS(&c[a[q]].meta, m[q], m[q] | (1ull << 63));
            for (int q = 2; q < 4; ++q) acc += ld_rlx(&c[a[q]].meta) ^ m[q];
        } else if (MODE >= 2) {
            for (int q = 0; q < 2; ++q) {
                const uint32_t si = (uint32_t)(mix(a[q] >> sshift) & smask);
                acc += atomicCAS(&st[si], s[q], s[q] | (1ull << 63));
            }
            for (int q = 2; q < 4; ++q) {
                const uint32_t si = (uint32_t)(mix(a[q] >> sshift) & smask);
                acc += ld_rlx(&st[si]) ^ s[q];
            }
        }
        for (int q = 0; q < 2; ++q) stv2(&c[a[q]], v[q] + 1, (m[q] + 1) & 0x7fffffffull);
        if (MODE >= 2) {
            if (MODE == 2) asm volatile("fence.acq_rel.gpu;" ::: "memory");
            for (int q = 0; q < 2; ++q) {
                const uint32_t si = (uint32_t)(mix(a[q] >> sshift) & smask);
                asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(&st[si]), "l"((s[q] + 1) & 0x7fffffffull)
                             : "memory");
            }
        }
    }
    if (acc == 42) *sink = acc;
}

struct Ent { unsigned long long addr, value, ts; };

__global__ void gen_log(Ent* e, uint64_t n, uint64_t W, uint64_t seed) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
        e[i] = Ent{mix(seed + i) % W, i * 7 + 1, seed + (i >> 1) + 1};
}
__global__ void ap_amax(Cell* c, const Ent* e, uint64_t n) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
        const Ent x = e[i];
        const unsigned long long old = atomicMax(&c[x.addr].meta, x.ts);
        if (old < x.ts) c[x.addr].value = x.value;
    }
}
__global__ void ap_blind(Cell* c, const Ent* e, uint64_t n) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
        const Ent x = e[i];
        stv2(&c[x.addr], x.value, x.ts);
    }
}
__device__ __forceinline__ void exch128(Cell* p, unsigned long long v, unsigned long long m, unsigned long long& ov,
                                        unsigned long long& om) {
    asm volatile("{\n\t.reg .b128 d, s;\n\tmov.b128 s, {%2, %3};\n\tatom.relaxed.gpu.global.exch.b128 d, [%4], s;\n\t"
                 "mov.b128 {%0, %1}, d;\n\t}"
                 : "=l"(ov), "=l"(om) : "l"(v), "l"(m), "l"(p) : "memory");
}
// max-register by exchange: swap the entry in; a displaced fresher {value, ts}
// is swapped back until the hand holds the smaller one
__global__ void ap_exch(Cell* c, const Ent* e, uint64_t n, unsigned long long* extra) {
    unsigned long long nx = 0;
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
        const Ent x = e[i];
        unsigned long long hv = x.value, hm = x.ts, ov, om;
        exch128(&c[x.addr], hv, hm, ov, om);
        while (om > hm || (om == hm && ov > hv)) {
            hv = ov; hm = om; ++nx;
            exch128(&c[x.addr], hv, hm, ov, om);
        }
    }
    if (nx) atomicAdd(extra, nx);
}
__global__ void ap_t1(unsigned long long* t, uint32_t mask, const Ent* e, uint64_t n) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
        const Ent x = e[i];
        atomicMax(&t[mix(x.addr) & mask], x.ts);
    }
}
__global__ void ap_t2(Cell* c, const unsigned long long* t, uint32_t mask, const Ent* e, uint64_t n,
                      unsigned long long* slow) {
    unsigned long long ns = 0;
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
        const Ent x = e[i];
        if (t[mix(x.addr) & mask] == x.ts) stv2(&c[x.addr], x.value, x.ts);
        else ++ns;
    }
    if (ns) atomicAdd(slow, ns);
}

int main() {
    const uint64_t W = 1ull << 27, N = 1ull << 20;
    Cell* c; unsigned long long *st, *sink;
    cudaMalloc(&c, W * sizeof(Cell)); cudaMemset(c, 0, W * sizeof(Cell)); cudaMalloc(&sink, 16);
    cudaMalloc(&st, (1ull << 24) * 8); cudaMemset(st, 0, (1ull << 24) * 8);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    auto timeit = [&](auto&& f) {
        float best = 1e9;
        for (int rep = 0; rep < 6; ++rep) {
            cudaEventRecord(a); f(rep); cudaEventRecord(b); cudaEventSynchronize(b);
            float ms; cudaEventElapsedTime(&ms, a, b);
            if (rep && ms < best) best = ms;
        }
        return best;
    };
    const char* names[] = {"floor (ld a0,a1 + st a0,a1)", "cell locks (today's shape)", "stripe table (acq/fence)",
                           "stripe table (no ordering)"};
    for (int sbits : {21, 22, 23, 24})
        for (int bps : {1, 2, 4}) {
            for (int mode = 0; mode < 4; ++mode) {
                if (mode < 2 && sbits != 21) continue;
                const uint32_t smask = (1u << sbits) - 1;
                float ms = timeit([&](int rep) {
                    const uint64_t seed = 1000 + rep * N * 8;
                    switch (mode) {
                        case 0: tx<0><<<148 * bps, 256>>>(c, st, W, smask, 0, N, seed, sink); break;
                        case 1: tx<1><<<148 * bps, 256>>>(c, st, W, smask, 0, N, seed, sink); break;
                        case 2: tx<2><<<148 * bps, 256>>>(c, st, W, smask, 0, N, seed, sink); break;
                        case 3: tx<3><<<148 * bps, 256>>>(c, st, W, smask, 0, N, seed, sink); break;
                    }
                });
                printf("tx  stripes 2^%d (%3d MiB)  CTAs/SM %d  %-32s %.4f ms  %.2f G tx/s\n", sbits,
                       (int)((8ull << sbits) >> 20), bps, names[mode], ms, N / ms / 1e6);
            }
        }
    cudaError_t err = cudaDeviceSynchronize();
    if (err != cudaSuccess) { printf("error %s\n", cudaGetErrorString(err)); return 1; }
    Ent* log; cudaMalloc(&log, 32 * N * sizeof(Ent));
    unsigned long long* slow; cudaMalloc(&slow, 8);
    gen_log<<<1184, 256>>>(log, 32 * N, W, 777);
    for (int bps : {1, 2, 4, 8}) {
        float m1 = timeit([&](int rep) { ap_amax<<<148 * bps, 256>>>(c, log + (rep % 32) * N, N); });
        float m2 = timeit([&](int rep) { ap_blind<<<148 * bps, 256>>>(c, log + (rep % 32) * N, N); });
        float m4 = timeit([&](int rep) { ap_exch<<<148 * bps, 256>>>(c, log + (rep % 32) * N, N, slow); });
        printf("apply CTAs/SM %d  exch128 %.4f ms (%.1f G/s)\n", bps, m4, N / m4 / 1e6);
        for (int tb : {21, 22}) {
            const uint32_t mask = (1u << tb) - 1;
            float m3 = timeit([&](int rep) {
                ap_t1<<<148 * bps, 256>>>(st, mask, log + (rep % 32) * N, N);
                ap_t2<<<148 * bps, 256>>>(c, st, mask, log + (rep % 32) * N, N, slow);
            });
            printf("apply CTAs/SM %d  table 2^%d: amax %.4f ms (%.1f G/s)  blind %.4f ms (%.1f G/s)  table %.4f ms (%.1f G/s)\n",
                   bps, tb, m1, N / m1 / 1e6, m2, N / m2 / 1e6, m3, N / m3 / 1e6);
        }
    }
    err = cudaDeviceSynchronize();
    if (err != cudaSuccess) { printf("error %s\n", cudaGetErrorString(err)); return 1; }
    return 0;
}
