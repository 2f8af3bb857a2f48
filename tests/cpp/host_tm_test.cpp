// host_tm_test.cpp — CPU checks of the host guest TM (include/hetm_b200/host_tm.hpp)
// against SPEC.md:123-170 examples and its invariants:
//   begin on a fresh system -> startTs 0; after one update commit -> 1
//   read-your-writes, zero-init reads, last write wins, write implies read
//   read-only commit returns startTs and logs nothing; first update ts = 1 with |writeSet|
//   entries
//   stale read after a concurrent commit aborts (opacity)
//   multi-threaded bank: sum invariant, unique ts, per-thread ts order,
//   log completeness (ts-order replay of the log == replica)
#include <algorithm>
#include <cstdio>
#include <thread>
#include <unordered_set>
#include <vector>

#include "hetm_b200/host_tm.hpp"

using namespace hetm::b200;

#define EXPECT(c)                                                   \
    do {                                                            \
        if (!(c)) {                                                 \
            std::printf("FAILED %s:%d: %s\n", __FILE__, __LINE__, #c); \
            return 1;                                               \
        }                                                           \
    } while (0)

int main() {
    {  // SPEC examples, single thread
        std::vector<uint64_t> mem(64, 0);
        HostStm stm(mem.data(), mem.size(), 10);
        WriteLog log(1);
        stm.setCommitCallback([&](int t, std::span<const hetm_log_entry> es) { log.append(t, es); });
        HostStm::Tx tx;
        TM_begin(stm, tx, 0);
        EXPECT(tx.rv == 0);
        EXPECT(TM_read(stm, tx, 7) == 0);                  // zero-init
        EXPECT(TM_commit(stm, tx) == 0 && log.entryCount(0) == 0);  // read-only: startTs, no log
        TM_begin(stm, tx, 0);
        TM_write(stm, tx, 5, 9);
        EXPECT(TM_read(stm, tx, 5) == 9);                  // read-your-writes
        TM_write(stm, tx, 5, 11);                          // last write wins
        TM_write(stm, tx, 6, 1);
        EXPECT(tx.reads.size() == 2);                      // writes imply reads
        EXPECT(TM_commit(stm, tx) == 1);
        EXPECT(mem[5] == 11 && mem[6] == 1 && log.entryCount(0) == 2);
        for (auto& e : log.allEntries()) EXPECT(e.ts == 1);
        TM_begin(stm, tx, 0);
        EXPECT(tx.rv == 1);
        // opacity: tx A reads 5, B commits a write to 5, A's next read of 5's lock sees a newer version
        HostStm::Tx a, b;
        TM_begin(stm, a, 0);
        EXPECT(TM_read(stm, a, 5) == 11);
        TM_begin(stm, b, 0);
        TM_write(stm, b, 5, 12);
        EXPECT(TM_commit(stm, b) == 2);
        bool aborted = false;
        try {
            TM_write(stm, a, 6, 3);  // 6's version (1) <= rv; commit must fail validation on 5
            TM_commit(stm, a);
        } catch (const TxAbort&) {
            aborted = true;
        }
        EXPECT(aborted && mem[5] == 12 && mem[6] == 1);
        bool oob = false;
        try {
            TM_begin(stm, tx, 0);
            TM_read(stm, tx, 64);
        } catch (const HostOutOfBounds&) {
            oob = true;
        }
        EXPECT(oob);
    }
    {  // multi-threaded bank transfers
        const uint64_t W = 4096;
        const int T = 8, N = 20000;
        std::vector<uint64_t> mem(W, 1000);
        HostStm stm(mem.data(), W, 12);
        WriteLog log(T);
        stm.setCommitCallback([&](int t, std::span<const hetm_log_entry> es) { log.append(t, es); });
        std::vector<std::thread> th;
        for (int t = 0; t < T; ++t)
            th.emplace_back([&, t] {
                uint64_t s = 0x1234 + t;
                for (int k = 0; k < N; ++k) {
                    s = s * 6364136223846793005ull + 1442695040888963407ull;
                    const uint64_t a = (s >> 20) % 64, b = (s >> 40) % W, amt = s % 7 + 1;  // hot words 0..63
                    if (a == b) continue;
                    stm.atomically(t, [&](HostStm::Tx& tx) {
                        const uint64_t x = TM_read(stm, tx, a), y = TM_read(stm, tx, b);
                        TM_write(stm, tx, a, x - amt);
                        TM_write(stm, tx, b, y + amt);
                    });
                }
            });
        for (auto& x : th) x.join();
        uint64_t sum = 0;
        for (uint64_t v : mem) sum += v;
        EXPECT(sum == 1000 * W);
        std::vector<uint64_t> replay(W, 1000);
        auto all = log.allEntries();
        std::unordered_set<uint64_t> ts_seen;
        for (int t = 0; t < T; ++t) {  // ts-ordered within a thread (write_log.hpp:27-28)
            std::vector<hetm_log_entry> es(log.entryCount(t));
            log.slice(t, 0, es.size(), es.data());
            for (std::size_t i = 1; i < es.size(); ++i) EXPECT(es[i - 1].ts <= es[i].ts);
        }
        std::stable_sort(all.begin(), all.end(), [](auto& x, auto& y) { return x.ts < y.ts; });
        for (std::size_t i = 0; i + 1 < all.size(); i += 2) {  // 2 entries per tx share one unique ts
            EXPECT(all[i].ts == all[i + 1].ts);
            EXPECT(ts_seen.insert(all[i].ts).second);
        }
        for (auto& e : all) replay[e.addr] = e.value;
        EXPECT(replay == mem);  // log completeness
        std::printf("{\"host_tm_test\": \"ok\", \"commits\": %zu, \"aborts\": %llu}\n", all.size() / 2,
                    (unsigned long long)stm.aborts());
    }
    return 0;
}
