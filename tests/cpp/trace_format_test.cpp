// trace_format_test.cpp — include/hetm_b200/trace.hpp on the CPU: 8 threads
// append concurrently (one global seq, per-thread program order), the trace
// is dumped, loaded back and compared bit-exactly, and a
// truncated file is rejected.  Usage: trace_format_test <path>; prints the
// event count.  Exit 0 = pass.
#include <cstdio>
#include <cstring>
#include <thread>
#include <vector>

#include "hetm_b200/trace.hpp"

using namespace hetm::b200;

int main(int argc, char** argv) {
    if (argc < 2) return 2;
    const std::string path = argv[1];
    Trace t(4096, "{\"threads\": 8}");
    t.beginRound(0);
    std::vector<std::thread> th;
    for (int w = 0; w < 8; ++w)
        th.emplace_back([&t, w] {
            for (uint64_t k = 0; k < 1000; ++k)
                t.append(0, (uint8_t)(k % 3), (uint64_t)w << 40 | k, k * 7 % 4096, k);
        });
    for (auto& x : th) x.join();
    const auto a = t.events();
    t.dump(path);
    const Trace u = Trace::load(path);
    const auto b = u.events();
    if (a.size() != b.size() || std::memcmp(a.data(), b.data(), a.size() * sizeof(hetm_trace_event)) != 0) {
        std::printf("round trip mismatch\n");
        return 1;
    }
    if (u.sizeWords() != 4096 || u.config() != "{\"threads\": 8}") {
        std::printf("header mismatch: %s\n", u.header().c_str());
        return 1;
    }
    // a truncated record must be rejected
    const std::string bad = path + ".bad";
    {
        FILE* f = std::fopen(path.c_str(), "rb");
        FILE* g = std::fopen(bad.c_str(), "wb");
        std::vector<char> buf(1 << 20);
        size_t n = std::fread(buf.data(), 1, buf.size(), f);
        std::fwrite(buf.data(), 1, n - 7, g);
        std::fclose(f);
        std::fclose(g);
    }
    bool threw = false;
    try {
        (void)Trace::load(bad);
    } catch (const std::exception&) {
        threw = true;
    }
    std::remove(bad.c_str());
    if (!threw) {
        std::printf("truncated trace accepted\n");
        return 1;
    }
    std::printf("events %zu\n", a.size());
    return 0;
}
