// host_order_probe.cpp — does the ORDER of the delta records change the host
// merge scatter? (not product code).  2^21 {loc, value} records over the lower
// 512 MiB of a 1 GiB THP replica (a cfg2 round's device write set), scattered
// by T threads claiming 8K-record blocks (the product's worker pool), with a
// prefetch-for-write distance of 64, in three orders:
//   random    records in arbitrary order
//   bucket    grouped by 256 contiguous address ranges (the product's emit)
//   sorted    ascending address
// Fresh addresses every repetition.
//   g++ -O3 -pthread -o build/host_order_probe tools/host_order_probe.cpp
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

struct Rec { uint32_t loc; uint64_t value; };

int main() {
    const uint64_t W = 1ull << 27, span = W / 2, n = 1ull << 21, block = 8192;
    uint64_t* host = static_cast<uint64_t*>(mmap(nullptr, W * 8, PROT_READ | PROT_WRITE,
                                                 MAP_PRIVATE | MAP_ANONYMOUS, -1, 0));
    madvise(host, W * 8, MADV_HUGEPAGE);
    memset(host, 1, W * 8);
    const unsigned hc = std::thread::hardware_concurrency();
    const int T = hc > 1 ? (int)hc - 1 : 1;
    printf("hardware_concurrency %u, threads %d\n", hc, T);
    std::mt19937_64 g(11);
    const int kReps = 8;
    for (int order = 0; order < 3; ++order) {
        double best = 1e9, sum = 0;
        for (int rep = 0; rep < kReps; ++rep) {
            std::vector<Rec> r(n);
            for (uint64_t i = 0; i < n; ++i) r[i] = Rec{(uint32_t)(g() % span), i};
            if (order == 1)
                std::stable_sort(r.begin(), r.end(), [](const Rec& a, const Rec& b) { return (a.loc >> 19) < (b.loc >> 19); });
            if (order == 2) std::sort(r.begin(), r.end(), [](const Rec& a, const Rec& b) { return a.loc < b.loc; });
            std::atomic<uint64_t> next{0};
            auto t0 = std::chrono::steady_clock::now();
            std::vector<std::thread> th;
            for (int t = 0; t < T; ++t)
                th.emplace_back([&] {
                    for (;;) {
                        const uint64_t a = next.fetch_add(block);
                        if (a >= n) break;
                        const uint64_t b = std::min(n, a + block);
                        for (uint64_t i = a; i < b; ++i) {
                            if (i + 64 < b) __builtin_prefetch(&host[r[i + 64].loc], 1, 0);
                            host[r[i].loc] = r[i].value;
                        }
                    }
                });
            for (auto& x : th) x.join();
            const double ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
            if (rep) { best = std::min(best, ms); sum += ms; }
        }
        printf("%-7s best %.3f ms  mean %.3f ms  (%.0f M words/s best)\n",
               order == 0 ? "random" : order == 1 ? "bucket" : "sorted", best, sum / (kReps - 1), n / best / 1e3);
    }
    return 0;
}
