// apply_probe.cu — validateChunk(apply) design probe (not product code).
// Compares, on random 16-B word cells {value, meta}:
//   v0  returning atomicMax on meta + dependent value store + restore queue (round-1 product)
//   v1  one returning 128-bit exchange {value, TS} per entry; collisions with a
//       TS of this round queue the fresher of the pair; fixup = RED.MAX + winner store
//   v2  blind 16-B store per entry (upper bound, not a correct apply)
//   v3  RED.MAX on meta only (upper bound, not a correct apply)
// and checks v1 == v0 bit for bit on the final cells.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o build/apply_probe tools/apply_probe.cu
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>
#include <algorithm>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s:%d %s: %s\n", __FILE__, __LINE__, #x, cudaGetErrorString(e)); exit(1); } } while (0)

struct alignas(16) Cell { uint64_t value; unsigned long long meta; };
struct Entry { uint64_t addr, value, ts; };
constexpr unsigned long long kTag = 1ull << 62;

__host__ __device__ __forceinline__ uint64_t mix(uint64_t x) {
    x ^= x >> 33; x *= 0xff51afd7ed558ccdULL; x ^= x >> 33; x *= 0xc4ceb9fe1a85ec53ULL; x ^= x >> 33; return x;
}

__global__ void gen_log(Entry* log, uint64_t n, uint64_t W, uint64_t ts0, uint64_t seed, uint32_t hot_pct) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t h = mix(seed * 0x9e3779b97f4a7c15ull + i);
        uint64_t a = h % W;
        if ((h >> 40) % 100 < hot_pct) a = (mix(h) % 65536) * (W / 65536);  // hot set of 2^16 words
        log[i] = Entry{a, mix(h + 1), ts0 + 1 + (mix(h + 2) % n)};  // ts: random permutation-ish order, > ts0
    }
}

__device__ __forceinline__ void xchg128(Cell* c, uint64_t v, unsigned long long m, uint64_t& ov, unsigned long long& om) {
    asm volatile("{\n\t.reg .b128 d, s;\n\tmov.b128 s, {%2, %3};\n\tatom.relaxed.gpu.global.exch.b128 d, [%4], s;\n\tmov.b128 {%0, %1}, d;\n\t}"
                 : "=l"(ov), "=l"(om) : "l"(v), "l"(m), "l"(c) : "memory");
}
__device__ __forceinline__ void st128(Cell* c, uint64_t v, unsigned long long m) {
    asm volatile("{\n\t.reg .b128 t;\n\tmov.b128 t, {%1, %2};\n\tst.relaxed.gpu.global.b128 [%0], t;\n\t}" ::"l"(c), "l"(v), "l"(m) : "memory");
}

struct Ctr { unsigned long long restore_n, fix_n, conflict; };

template <int U>
__global__ void __launch_bounds__(256) apply_v0(Cell* cells, const Entry* __restrict__ log, uint64_t n, uint64_t floor_,
                                                const unsigned long long* rs, Ctr* ctr, unsigned long long* restore) {
    unsigned conflict = 0;
    const uint64_t span = (uint64_t)gridDim.x * blockDim.x * U;
    for (uint64_t i0 = (uint64_t)blockIdx.x * blockDim.x * U + threadIdx.x; i0 < n; i0 += span) {
        Entry e[U]; unsigned long long old[U];
#pragma unroll
        for (int u = 0; u < U; ++u) { const uint64_t i = i0 + u * blockDim.x; e[u] = i < n ? log[i] : Entry{0, 0, 0}; }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            old[u] = ~0ull;
            if (i0 + u * blockDim.x >= n) continue;
            const uint64_t bit = e[u].addr >> 7;
            conflict |= (unsigned)((rs[bit >> 6] >> (bit & 63)) & 1ull);
            old[u] = atomicMax(&cells[e[u].addr].meta, kTag | e[u].ts);
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            if (old[u] >= (kTag | e[u].ts)) continue;
            cells[e[u].addr].value = e[u].value;
            if ((old[u] & kTag) && (old[u] & ~kTag) > floor_) {
                const unsigned long long k = atomicAdd(&ctr->restore_n, 1ull);
                if (k < (1u << 20)) restore[k] = i0 + u * blockDim.x;
            }
        }
    }
    if (__any_sync(~0u, conflict) && (threadIdx.x & 31) == 0) atomicOr((unsigned*)&ctr->conflict, 1u);
}
__global__ void restore_v0(Cell* cells, const Entry* log, uint64_t n, Ctr* ctr, const unsigned long long* restore) {
    const unsigned long long m = ctr->restore_n;
    const bool full = m > (1u << 20);
    const uint64_t cnt = full ? n : m;
    for (uint64_t j = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; j < cnt; j += (uint64_t)gridDim.x * blockDim.x) {
        const Entry e = log[full ? j : restore[j]];
        if (*(volatile unsigned long long*)&cells[e.addr].meta == (kTag | e.ts)) cells[e.addr].value = e.value;
    }
}

template <int U>
__global__ void __launch_bounds__(256) apply_v1(Cell* cells, const Entry* __restrict__ log, uint64_t n, uint64_t floor_,
                                                const unsigned long long* rs, Ctr* ctr, Entry* fix) {
    unsigned conflict = 0;
    const uint64_t span = (uint64_t)gridDim.x * blockDim.x * U;
    for (uint64_t i0 = (uint64_t)blockIdx.x * blockDim.x * U + threadIdx.x; i0 < n; i0 += span) {
        Entry e[U]; uint64_t ov[U]; unsigned long long om[U];
#pragma unroll
        for (int u = 0; u < U; ++u) { const uint64_t i = i0 + u * blockDim.x; e[u] = i < n ? log[i] : Entry{0, 0, 0}; }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            om[u] = 0;
            if (i0 + u * blockDim.x >= n) continue;
            const uint64_t bit = e[u].addr >> 7;
            conflict |= (unsigned)((rs[bit >> 6] >> (bit & 63)) & 1ull);
            xchg128(&cells[e[u].addr], e[u].value, kTag | e[u].ts, ov[u], om[u]);
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const uint64_t ots = om[u] & ~kTag;
            if ((om[u] & kTag) && (ots > floor_ || ots >= e[u].ts)) {  // displaced a TS of this round (or a fresher one)
                const Entry c = ots > e[u].ts ? Entry{e[u].addr, ov[u], ots} : e[u];
                const unsigned long long k = atomicAdd(&ctr->fix_n, 1ull);
                fix[k] = c;
            }
        }
    }
    if (__any_sync(~0u, conflict) && (threadIdx.x & 31) == 0) atomicOr((unsigned*)&ctr->conflict, 1u);
}
__global__ void fix_max(Cell* cells, const Entry* fix, const Ctr* ctr) {
    const uint64_t m = *(volatile const unsigned long long*)&ctr->fix_n;
    for (uint64_t j = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; j < m; j += (uint64_t)gridDim.x * blockDim.x)
        atomicMax(&cells[fix[j].addr].meta, kTag | fix[j].ts);
}
__global__ void fix_store(Cell* cells, const Entry* fix, Ctr* ctr) {
    const uint64_t m = *(volatile unsigned long long*)&ctr->fix_n;
    for (uint64_t j = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; j < m; j += (uint64_t)gridDim.x * blockDim.x) {
        const Entry c = fix[j];
        if (*(volatile unsigned long long*)&cells[c.addr].meta == (kTag | c.ts)) cells[c.addr].value = c.value;
    }
}

// v4: first touch of a word this round (per a hashed filter of fbits bits,
// returning atomicOr in L2) stores {value, TS} blind; later touches and filter
// collisions go to the fix queue (RED.MAX + winner store after the launch).
template <int U>
__global__ void __launch_bounds__(256) apply_v4(Cell* cells, const Entry* __restrict__ log, uint64_t n, uint64_t floor_,
                                                const unsigned long long* rs, Ctr* ctr, Entry* fix,
                                                unsigned long long* filt, uint32_t fshift) {
    unsigned conflict = 0;
    const uint64_t span = (uint64_t)gridDim.x * blockDim.x * U;
    for (uint64_t i0 = (uint64_t)blockIdx.x * blockDim.x * U + threadIdx.x; i0 < n; i0 += span) {
        Entry e[U]; unsigned long long got[U], m[U];
#pragma unroll
        for (int u = 0; u < U; ++u) { const uint64_t i = i0 + u * blockDim.x; e[u] = i < n ? log[i] : Entry{0, 0, 0}; }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            m[u] = 0; got[u] = ~0ull;
            if (i0 + u * blockDim.x >= n) continue;
            const uint64_t bit = e[u].addr >> 7;
            conflict |= (unsigned)((rs[bit >> 6] >> (bit & 63)) & 1ull);
            const uint64_t h = (e[u].addr * 0x9e3779b97f4a7c15ull) >> fshift;  // 64 - fshift bits
            m[u] = 1ull << (h & 63);
            got[u] = atomicOr(&filt[h >> 6], m[u]);
        }
        bool slow[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            slow[u] = false;
            if (!m[u]) continue;
            if (!(got[u] & m[u])) st128(&cells[e[u].addr], e[u].value, kTag | e[u].ts);
            else slow[u] = true;
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const unsigned b = __ballot_sync(~0u, slow[u]);
            if (!b) continue;
            unsigned long long base = 0;
            if ((threadIdx.x & 31) == __ffs(b) - 1) base = atomicAdd(&ctr->fix_n, (unsigned long long)__popc(b));
            base = __shfl_sync(~0u, base, __ffs(b) - 1);
            if (slow[u]) fix[base + __popc(b & ((1u << (threadIdx.x & 31)) - 1))] = e[u];
        }
    }
    if (__any_sync(~0u, conflict) && (threadIdx.x & 31) == 0) atomicOr((unsigned*)&ctr->conflict, 1u);
}

template <int U>
__global__ void __launch_bounds__(256) apply_v2(Cell* cells, const Entry* __restrict__ log, uint64_t n) {
    const uint64_t span = (uint64_t)gridDim.x * blockDim.x * U;
    for (uint64_t i0 = (uint64_t)blockIdx.x * blockDim.x * U + threadIdx.x; i0 < n; i0 += span) {
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const uint64_t i = i0 + u * blockDim.x;
            if (i < n) { const Entry e = log[i]; st128(&cells[e.addr], e.value, kTag | e.ts); }
        }
    }
}
template <int U>
__global__ void __launch_bounds__(256) apply_v3(Cell* cells, const Entry* __restrict__ log, uint64_t n) {
    const uint64_t span = (uint64_t)gridDim.x * blockDim.x * U;
    for (uint64_t i0 = (uint64_t)blockIdx.x * blockDim.x * U + threadIdx.x; i0 < n; i0 += span) {
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const uint64_t i = i0 + u * blockDim.x;
            if (i < n) { const Entry e = log[i]; atomicMax(&cells[e.addr].meta, kTag | e.ts); }
        }
    }
}

int main(int argc, char** argv) {
    const int wl2 = argc > 1 ? atoi(argv[1]) : 27;
    const int nl2 = argc > 2 ? atoi(argv[2]) : 20;
    const uint32_t hot = argc > 3 ? atoi(argv[3]) : 0;
    const uint64_t W = 1ull << wl2, n = 1ull << nl2;
    int sms = 0;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
    Cell *c0, *c1;
    Entry *log, *fix;
    unsigned long long *rs, *restore;
    Ctr* ctr;
    CK(cudaMalloc(&c0, W * 16));
    CK(cudaMalloc(&c1, W * 16));
    CK(cudaMalloc(&log, n * sizeof(Entry)));
    CK(cudaMalloc(&fix, n * sizeof(Entry)));
    CK(cudaMalloc(&rs, (W / 128 / 8) + 64));
    CK(cudaMalloc(&restore, 8u << 20));
    CK(cudaMalloc(&ctr, sizeof(Ctr)));
    CK(cudaMemset(c0, 0, W * 16));
    CK(cudaMemset(c1, 0, W * 16));
    Cell *c2, *c3;
    CK(cudaMalloc(&c2, W * 16));
    CK(cudaMalloc(&c3, W * 16));
    CK(cudaMemset(c2, 0, W * 16));
    CK(cudaMemset(c3, 0, W * 16));
    uint32_t fbits[2];
    fbits[0] = std::min<uint32_t>(29, std::max<uint32_t>(23, nl2 + 5));  // 32 bits per entry
    fbits[1] = std::min<uint32_t>(29, std::max<uint32_t>(23, nl2 + 3));  // 8 bits per entry
    unsigned long long* filt;
    CK(cudaMalloc(&filt, (1ull << 29) / 8));
    double t4[2] = {0, 0}, tclr[2] = {0, 0};
    CK(cudaMemset(rs, 0, (W / 128 / 8) + 64));
    cudaEvent_t a, b;
    CK(cudaEventCreate(&a));
    CK(cudaEventCreate(&b));
    const int reps = 8;
    double t[6] = {0};
    for (int r = 0; r < reps; ++r) {
        const uint64_t ts0 = (uint64_t)r * n * 2, floor_ = ts0;
        gen_log<<<sms * 8, 256>>>(log, n, W, ts0, 1000 + r, hot);
        auto grid = [&](int U, int bps) { uint64_t g = (n + 256 * U - 1) / (256 * U); uint64_t cap = (uint64_t)sms * bps; return (unsigned)(g < cap ? g : cap); };
        float ms;
        // v0
        CK(cudaMemset(ctr, 0, sizeof(Ctr)));
        CK(cudaEventRecord(a));
        apply_v0<4><<<grid(4, 1), 256>>>(c0, log, n, floor_, rs, ctr, restore);
        restore_v0<<<2 * sms, 256>>>(c0, log, n, ctr, restore);
        CK(cudaEventRecord(b));
        CK(cudaEventSynchronize(b));
        CK(cudaEventElapsedTime(&ms, a, b));
        if (r) t[0] += ms;
        // v1 on c1 (the checked copy), same log
        CK(cudaMemset(ctr, 0, sizeof(Ctr)));
        CK(cudaEventRecord(a));
        apply_v1<4><<<grid(4, 1), 256>>>(c1, log, n, floor_, rs, ctr, fix);
        fix_max<<<2 * sms, 256>>>(c1, fix, ctr);
        fix_store<<<2 * sms, 256>>>(c1, fix, ctr);
        CK(cudaEventRecord(b));
        CK(cudaEventSynchronize(b));
        CK(cudaEventElapsedTime(&ms, a, b));
        if (r) t[1] += ms;
        Ctr h;
        CK(cudaMemcpy(&h, ctr, sizeof h, cudaMemcpyDeviceToHost));
        if (r == reps - 1) printf("  v1 fix queue: %llu of %llu entries\n", h.fix_n, (unsigned long long)n);
        // v4 on c2, filter cleared per round (the clear is timed separately)
        for (int fi = 0; fi < 2; ++fi) {
            const uint32_t fb = fbits[fi];
            CK(cudaEventRecord(a));
            CK(cudaMemsetAsync(filt, 0, (1ull << fb) / 8));
            CK(cudaEventRecord(b));
            CK(cudaEventSynchronize(b));
            CK(cudaEventElapsedTime(&ms, a, b));
            if (r) tclr[fi] += ms;
            CK(cudaMemset(ctr, 0, sizeof(Ctr)));
            Cell* dst = fi == 0 ? c2 : c3;
            CK(cudaEventRecord(a));
            apply_v4<4><<<grid(4, 1), 256>>>(dst, log, n, floor_, rs, ctr, fix, filt, 64 - fb);
            fix_max<<<2 * sms, 256>>>(dst, fix, ctr);
            fix_store<<<2 * sms, 256>>>(dst, fix, ctr);
            CK(cudaEventRecord(b));
            CK(cudaEventSynchronize(b));
            CK(cudaEventElapsedTime(&ms, a, b));
            if (r) t4[fi] += ms;
            CK(cudaMemcpy(&h, ctr, sizeof h, cudaMemcpyDeviceToHost));
            if (r == reps - 1) printf("  v4 filter 2^%u bits: fix queue %llu of %llu entries\n", fb, h.fix_n, (unsigned long long)n);
        }
    }
    // correctness: c0 (v0) == c1 (v1)
    {
        std::vector<Cell> h0(1 << 20), h1(1 << 20);
        uint64_t bad = 0;
        for (uint64_t off = 0; off < W; off += h0.size()) {
            const uint64_t m = std::min<uint64_t>(h0.size(), W - off);
            CK(cudaMemcpy(h0.data(), c0 + off, m * 16, cudaMemcpyDeviceToHost));
            CK(cudaMemcpy(h1.data(), c1 + off, m * 16, cudaMemcpyDeviceToHost));
            for (uint64_t i = 0; i < m; ++i)
                if (h0[i].value != h1[i].value || h0[i].meta != h1[i].meta) ++bad;
        }
        printf("  v0 vs v1 cells differing: %llu\n", (unsigned long long)bad);
        for (Cell* cx : {c2, c3}) {
            bad = 0;
            for (uint64_t off = 0; off < W; off += h0.size()) {
                const uint64_t m = std::min<uint64_t>(h0.size(), W - off);
                CK(cudaMemcpy(h0.data(), c0 + off, m * 16, cudaMemcpyDeviceToHost));
                CK(cudaMemcpy(h1.data(), cx + off, m * 16, cudaMemcpyDeviceToHost));
                for (uint64_t i = 0; i < m; ++i)
                    if (h0[i].value != h1[i].value || h0[i].meta != h1[i].meta) ++bad;
            }
            printf("  v0 vs v4 cells differing: %llu\n", (unsigned long long)bad);
        }
        for (int fi = 0; fi < 2; ++fi)
            printf("W=2^%d n=2^%d hot=%u%%  v4 filter(2^%u bits)+blind st.b128+fix %8.4f ms  %6.2f G entries/s  (filter clear %.4f ms)\n",
                   wl2, nl2, hot, fbits[fi], t4[fi] / (reps - 1), n / (t4[fi] / (reps - 1)) / 1e6, tclr[fi] / (reps - 1));
    }
    // upper bounds
    for (int r = 0; r < reps; ++r) {
        const uint64_t ts0 = (uint64_t)(reps + r) * n * 2;
        gen_log<<<sms * 8, 256>>>(log, n, W, ts0, 5000 + r, hot);
        float ms;
        unsigned g4 = (unsigned)std::min<uint64_t>((n + 1023) / 1024, (uint64_t)sms * 2);
        CK(cudaEventRecord(a));
        apply_v2<4><<<g4, 256>>>(c1, log, n);
        CK(cudaEventRecord(b));
        CK(cudaEventSynchronize(b));
        CK(cudaEventElapsedTime(&ms, a, b));
        if (r) t[2] += ms;
        CK(cudaEventRecord(a));
        apply_v3<4><<<g4, 256>>>(c1, log, n);
        CK(cudaEventRecord(b));
        CK(cudaEventSynchronize(b));
        CK(cudaEventElapsedTime(&ms, a, b));
        if (r) t[3] += ms;
        // v1 again on uniquely fresh ts (timing on c1 after the bounds: every entry wins)
        CK(cudaMemset(ctr, 0, sizeof(Ctr)));
        gen_log<<<sms * 8, 256>>>(log, n, W, ts0 + n, 7000 + r, hot);
        unsigned g1 = (unsigned)std::min<uint64_t>((n + 1023) / 1024, (uint64_t)sms);
        CK(cudaEventRecord(a));
        apply_v1<4><<<g1 * 2 > (unsigned)sms * 2 ? sms * 2 : g1 * 2, 256>>>(c1, log, n, ts0 + n, rs, ctr, fix);
        fix_max<<<2 * sms, 256>>>(c1, fix, ctr);
        fix_store<<<2 * sms, 256>>>(c1, fix, ctr);
        CK(cudaEventRecord(b));
        CK(cudaEventSynchronize(b));
        CK(cudaEventElapsedTime(&ms, a, b));
        if (r) t[4] += ms;
        CK(cudaMemset(ctr, 0, sizeof(Ctr)));
        gen_log<<<sms * 8, 256>>>(log, n, W, ts0 + 3 * n, 9000 + r, hot);
        CK(cudaEventRecord(a));
        apply_v1<8><<<(unsigned)std::min<uint64_t>((n + 2047) / 2048, (uint64_t)sms), 256>>>(c1, log, n, ts0 + 3 * n, rs, ctr, fix);
        fix_max<<<2 * sms, 256>>>(c1, fix, ctr);
        fix_store<<<2 * sms, 256>>>(c1, fix, ctr);
        CK(cudaEventRecord(b));
        CK(cudaEventSynchronize(b));
        CK(cudaEventElapsedTime(&ms, a, b));
        if (r) t[5] += ms;
    }
    const char* names[6] = {"v0 atomicMax+store+restore (1 CTA/SM, U4)", "v1 exch128+fix (1 CTA/SM, U4)",
                            "v2 blind st.b128 (bound)", "v3 RED.MAX only (bound)", "v1 exch128+fix (2 CTA/SM, U4)",
                            "v1 exch128+fix (1 CTA/SM, U8)"};
    for (int k = 0; k < 6; ++k) {
        const double ms = t[k] / (reps - 1);
        printf("W=2^%d n=2^%d hot=%u%%  %-44s %8.4f ms  %6.2f G entries/s  %7.1f GB/s alg (120 B)\n", wl2, nl2, hot,
               names[k], ms, n / ms / 1e6, 120.0 * n / ms / 1e6);
    }
    return 0;
}
