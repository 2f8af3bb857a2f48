// dispatch_test.cpp — include/hetm_b200/dispatch.hpp on the CPU
// (SPEC.md:479-487 examples; exactly-once consumption):
//   * batchSize-1 queued -> no batch; batchSize queued -> exactly batchSize, FIFO;
//   * 8 producers x 10000 requests, the controller polling concurrently:
//     every request is dequeued exactly once, batches are exactly batchSize
//     except the max-wait tail;
//   * the max-wait knob releases a partial batch only after the wait.
// Exit 0 = pass (one line "ok").
#include <atomic>
#include <cstdio>
#include <thread>
#include <vector>

#include "hetm_b200/dispatch.hpp"

using namespace hetm::b200;

#define CHECK(c)                                                   \
    do {                                                           \
        if (!(c)) {                                                \
            std::printf("FAIL %s:%d %s\n", __FILE__, __LINE__, #c); \
            return 1;                                              \
        }                                                          \
    } while (0)

int main() {
    {
        DeviceQueue<hetm_bank_tx> q(4);
        std::vector<hetm_bank_tx> out;
        for (uint32_t i = 0; i < 3; ++i) q.submit(hetm_bank_tx{{i, i, i, i}, i});
        CHECK(!q.poll(out));  // batchSize - 1 -> none
        q.submit(hetm_bank_tx{{3, 3, 3, 3}, 3});
        CHECK(q.poll(out) && out.size() == 4);  // batchSize -> exactly batchSize
        for (uint32_t i = 0; i < 4; ++i) CHECK(out[i].amount == i);  // FIFO
        CHECK(q.size() == 0 && !q.poll(out));
    }
    {
        const uint64_t B = 97;
        DeviceQueue<hetm_bank_tx> q(B, std::chrono::microseconds(2000));
        std::atomic<int> producers{8};
        std::vector<std::thread> th;
        for (int p = 0; p < 8; ++p)
            th.emplace_back([&, p] {
                for (uint32_t k = 0; k < 10000; ++k) q.submit(hetm_bank_tx{{(uint32_t)p, k, 0, 0}, (uint64_t)p << 32 | k});
                producers.fetch_sub(1);
            });
        std::vector<uint8_t> seen(8 * 10000, 0);
        std::vector<hetm_bank_tx> out;
        uint64_t got = 0, partial = 0;
        std::vector<uint32_t> last(8, 0);
        bool fifo = true;
        while (got < 80000) {
            if (!q.poll(out)) {
                std::this_thread::yield();
                continue;
            }
            if (out.size() != B) ++partial;
            for (auto& r : out) {
                const uint64_t p = r.amount >> 32, k = r.amount & 0xffffffffu;
                CHECK(!seen[p * 10000 + k]);
                seen[p * 10000 + k] = 1;
                fifo &= k == 0 || k == last[p] + 1;  // each producer's requests stay in order
                last[p] = (uint32_t)k;
                ++got;
            }
        }
        for (auto& t : th) t.join();
        CHECK(got == 80000 && fifo);
        CHECK(partial <= 1);  // only the tail (80000 = 824 * 97 + 72) may be a partial batch
    }
    {
        DeviceQueue<hetm_bank_tx> q(10, std::chrono::microseconds(20000));
        std::vector<hetm_bank_tx> out;
        q.submit(hetm_bank_tx{{1, 2, 3, 4}, 5});
        CHECK(!q.poll(out));  // not yet
        std::this_thread::sleep_for(std::chrono::milliseconds(25));
        CHECK(q.poll(out) && out.size() == 1);  // the wait released the partial batch
    }
    std::printf("ok\n");
    return 0;
}
