// host_scatter_probe.cpp — host-side merge scatter throughput (not product code).
// Scatters n sorted {loc, value} records into a 1 GiB host replica with T
// threads, prefetch-for-write distance D, 4 KiB vs 2 MiB (THP) pages.
//   g++ -O3 -march=native -pthread -o build/host_scatter_probe tools/host_scatter_probe.cpp
#include <immintrin.h>
#include <sys/mman.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <random>
#include <thread>
#include <vector>

struct Rec { uint64_t loc, value; };

static uint64_t* alloc_replica(size_t bytes, bool huge) {
    void* p = mmap(nullptr, bytes, PROT_READ | PROT_WRITE, MAP_PRIVATE | MAP_ANONYMOUS, -1, 0);
    if (p == MAP_FAILED) return nullptr;
    madvise(p, bytes, huge ? MADV_HUGEPAGE : MADV_NOHUGEPAGE);
    memset(p, 1, bytes);
    return static_cast<uint64_t*>(p);
}

// D < 0: non-temporal 8-B stores (movnti), no RFO into the cache hierarchy
template <int D>
static void scatter(uint64_t* host, const Rec* r, uint64_t a, uint64_t b) {
    for (uint64_t i = a; i < b; ++i) {
        if (D < 0) {
            _mm_stream_si64(reinterpret_cast<long long*>(&host[r[i].loc]), (long long)r[i].value);
            continue;
        }
        if (D && i + D < b) __builtin_prefetch(&host[r[i + D].loc], 1, 0);
        host[r[i].loc] = r[i].value;
    }
    if (D < 0) _mm_sfence();
}

int main() {
    const uint64_t W = 1ull << 30, n = 1ull << 21;  // 8 GiB replica (cold lines); 2^21 records (a bank round's delta)
    // fresh sorted addresses every repetition: the merge of a round touches
    // lines no earlier round left in the LLC (a warm re-scatter is flattering)
    const int kReps = 6;
    std::vector<std::vector<Rec>> recs(kReps, std::vector<Rec>(n));
    std::mt19937_64 g(7);
    std::vector<uint64_t> locs(n);
    for (auto& rec : recs) {
        for (auto& l : locs) l = g() % W;
        std::sort(locs.begin(), locs.end());
        for (uint64_t i = 0; i < n; ++i) rec[i] = Rec{locs[i], i};
    }
    printf("hardware_concurrency %u\n", std::thread::hardware_concurrency());
    for (bool huge : {true}) {
        uint64_t* host = alloc_replica(W * 8, huge);
        for (int T : {15, 16}) {
            if ((unsigned)T > std::thread::hardware_concurrency()) continue;
            for (int D : {-1, 0, 32, 64}) {
                double best = 1e9;
                for (int rep = 0; rep < kReps; ++rep) {
                    const std::vector<Rec>& rec = recs[rep];
                    std::atomic<int> ready{0}, go{0};
                    std::vector<std::thread> th;
                    for (int w = 0; w < T; ++w)
                        th.emplace_back([&, w] {
                            ready.fetch_add(1);
                            while (!go.load(std::memory_order_acquire)) {}
                            const uint64_t a = n * w / T, b = n * (w + 1) / T;
                            switch (D) {
                                case -1: scatter<-1>(host, rec.data(), a, b); break;
                                case 0: scatter<0>(host, rec.data(), a, b); break;
                                case 8: scatter<8>(host, rec.data(), a, b); break;
                                case 16: scatter<16>(host, rec.data(), a, b); break;
                                case 32: scatter<32>(host, rec.data(), a, b); break;
                                case 64: scatter<64>(host, rec.data(), a, b); break;
                                default: scatter<128>(host, rec.data(), a, b); break;
                            }
                        });
                    while (ready.load() < T) {}
                    auto t0 = std::chrono::steady_clock::now();
                    go.store(1, std::memory_order_release);
                    for (auto& t : th) t.join();
                    const double ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
                    if (rep && ms < best) best = ms;
                }
                printf("%s T=%2d D=%2d: %.3f ms  %.0f M words/s\n", huge ? "THP " : "4KiB", T, D, best, n / best / 1e3);
            }
        }
        munmap(host, W * 8);
    }
    return 0;
}
