// host_mem_probe.cpp — host DRAM bandwidth of the GPU box (not product code):
// T threads streaming copy (read + write bytes) over 2 x 1 GiB THP buffers, and
// the random 8-B read-modify-write rate over a cold 8 GiB region (the merge
// scatter's pattern).  g++ -O3 -march=x86-64-v3 -pthread -o build/host_mem_probe tools/host_mem_probe.cpp
#include <sys/mman.h>

#include <atomic>
#include <chrono>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <random>
#include <thread>
#include <vector>

static void* thp(size_t bytes) {
    void* p = mmap(nullptr, bytes, PROT_READ | PROT_WRITE, MAP_PRIVATE | MAP_ANONYMOUS, -1, 0);
    madvise(p, bytes, MADV_HUGEPAGE);
    memset(p, 1, bytes);
    return p;
}

template <class F>
static double run(int T, F f) {
    std::atomic<int> ready{0}, go{0};
    std::vector<std::thread> th;
    for (int w = 0; w < T; ++w)
        th.emplace_back([&, w] {
            ready.fetch_add(1);
            while (!go.load()) {}
            f(w, T);
        });
    while (ready.load() < T) {}
    auto t0 = std::chrono::steady_clock::now();
    go.store(1);
    for (auto& t : th) t.join();
    return std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
}

int main() {
    const size_t N = 1ull << 30;
    char* a = static_cast<char*>(thp(N));
    char* b = static_cast<char*>(thp(N));
    for (int T : {8, 16}) {
        double best = 1e9;
        for (int r = 0; r < 4; ++r)
            best = std::min(best, run(T, [&](int w, int t) {
                const size_t lo = N * w / t, hi = N * (w + 1) / t;
                memcpy(b + lo, a + lo, hi - lo);
            }));
        printf("copy T=%2d: %.1f GB/s (read + write bytes)\n", T, 2.0 * N / best / 1e9);
    }
    const size_t W = 1ull << 30;  // 8 GiB of words, cold
    uint64_t* h = static_cast<uint64_t*>(thp(W * 8));
    const size_t n = 1ull << 22;
    std::vector<uint64_t> loc(n);
    std::mt19937_64 g(3);
    for (auto& l : loc) l = g() % W;
    for (int T : {8, 16}) {
        const double s = run(T, [&](int w, int t) {
            const size_t lo = n * w / t, hi = n * (w + 1) / t;
            for (size_t i = lo; i < hi; ++i) {
                if (i + 64 < hi) __builtin_prefetch(&h[loc[i + 64]], 1, 0);
                h[loc[i]] += 1;
            }
        });
        printf("random 8-B RMW T=%2d: %.0f M/s (%.1f GB/s of 128-B line traffic)\n", T, n / s / 1e6, n * 128.0 / s / 1e9);
    }
    return 0;
}
