// queue_round_test.cpp — engine rounds fed by the device submission queue
// (include/hetm_b200/dispatch.hpp): producer threads submit
// bank transfers (device half) while the engine's GPU-controller launches a
// batch whenever the queue holds batchSize of them; host workers commit
// through HostStm on the other half.  TEST INFRASTRUCTURE: every round is
// replayed on the CPU oracle — host log in ts order, then every launched
// batch in ticket order — and must equal both replicas bit-exactly; every
// submitted transfer is executed exactly once.
//   queue_round_test [rounds] [batch]     Exit 0 = pass; prints one JSON line.
#include <atomic>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <thread>
#include <vector>

#include "hetm_b200/capi.h"
#include "hetm_b200/dispatch.hpp"
#include "hetm_b200/engine.hpp"
#include "hetm_b200/host_tm.hpp"

extern "C" {  // oracle/hetm_oracle.h (test infrastructure)
typedef struct { uint32_t acct[4]; uint64_t amount; } orc_bank_tx;
typedef struct { uint64_t addr, value, ts; } orc_entry;
void orc_gen_bank_batch(uint64_t seed, uint64_t n, uint64_t lo, uint64_t span, orc_bank_tx* out);
void orc_bank_replay(uint64_t* s, uint64_t base, const orc_bank_tx* tx, const uint64_t* order, uint64_t n_order,
                     uint64_t* rs, uint64_t* ws, uint64_t* ch, uint64_t gran, uint64_t chunk);
uint64_t orc_order_by_ticket(const uint64_t* tickets, uint64_t n, uint64_t* order_out);
void orc_apply_log_ts_order(uint64_t* region, uint64_t base, const orc_entry* e, uint64_t n);
uint64_t orc_splitmix64(uint64_t x);
}

using namespace hetm::b200;

int main(int argc, char** argv) {
    const int rounds = argc > 1 ? std::atoi(argv[1]) : 5;
    const uint64_t B = argc > 2 ? std::strtoull(argv[2], nullptr, 10) : 4096;
    const uint64_t W = 1ull << 20, half = W / 2;
    hetm_dev_config cfg;
    hetm_dev_config_default(&cfg);
    cfg.size_words = W;
    cfg.flags = HETM_CFG_MERGE_DELTA;
    hetm_dev* dev = nullptr;
    if (int rc = hetm_dev_open(&cfg, &dev); rc != HETM_OK) {
        std::printf("open: %s\n", hetm_strerror(rc));
        return rc == HETM_ERR_NO_DEVICE ? 3 : 1;
    }
    check_rc(hetm_dev_register_kernel(dev, HETM_KERNEL_BANK), "register");
    uint64_t* host = nullptr;
    check_rc(hetm_host_alloc(W * 8, reinterpret_cast<void**>(&host)), "host_alloc");
    for (uint64_t i = 0; i < W; ++i) host[i] = 1000;
    check_rc(hetm_dev_upload(dev, HETM_REPLICA_DEV, 0, host, W), "upload");
    check_rc(hetm_dev_merge_commit(dev, host, nullptr), "merge");
    check_rc(hetm_dev_merge_wait(dev), "merge_wait");
    check_rc(hetm_dev_clear_round(dev, 0), "clear");
    const int T = 4;
    HostStm stm(host, W, 20);
    WriteLog log(T);
    stm.setCommitCallback([&](int t, std::span<const hetm_log_entry> es) { log.append(t, es); });
    EngineConfig ec;
    ec.keep_round_log = true;
    Engine eng(dev, stm, log, host, ec);
    DeviceQueue<hetm_bank_tx> q(B);
    std::vector<uint64_t> ref(host, host + W);
    bool ok = true;
    uint64_t submitted = 0, executed = 0, batches = 0;
    for (int r = 0; r < rounds && ok; ++r) {
        // two producers submit 2.5 batches' worth of transfers concurrently with the round
        std::vector<std::thread> prod;
        std::atomic<uint64_t> sub{0};
        for (int p = 0; p < 2; ++p)
            prod.emplace_back([&, p] {
                std::vector<orc_bank_tx> t(B * 5 / 4);
                orc_gen_bank_batch(9000 + 16 * r + p, t.size(), 0, half, t.data());
                for (auto& x : t) q.submit(reinterpret_cast<const hetm_bank_tx&>(x));
                sub += t.size();
            });
        for (auto& p : prod) p.join();  // the queue is full before the round; the tail waits for the next
        submitted += sub;
        std::vector<hetm_bank_tx> buf;
        std::vector<uint64_t> tk;
        std::vector<orc_bank_tx> round_tx;
        std::vector<uint64_t> round_tk;
        auto src = q.source(buf, tk);
        bool pending = false;  // buf / tk hold a launched batch not recorded yet
        auto record = [&] {
            if (!pending) return;
            round_tx.insert(round_tx.end(), reinterpret_cast<const orc_bank_tx*>(buf.data()),
                            reinterpret_cast<const orc_bank_tx*>(buf.data()) + buf.size());
            round_tk.insert(round_tk.end(), tk.begin(), tk.end());
            pending = false;
        };
        auto recording = [&](uint32_t k, Engine::Batch& b) {  // keep every launched batch for the replay
            record();
            pending = src(k, b);
            return pending;
        };
        auto worker = [&](int t, const RoundContext& ctx) -> uint64_t {
            uint64_t s = orc_splitmix64(31u * r + t + 1), done = 0;
            for (int k = 0; k < 800 && !ctx.stop.load(std::memory_order_relaxed); ++k) {
                uint64_t a[2];
                for (auto& x : a) {
                    s = orc_splitmix64(s);
                    x = half + s % half;
                }
                if (a[0] == a[1]) continue;
                stm.atomically(t, [&](HostStm::Tx& tx) {
                    const uint64_t x = TM_read(stm, tx, a[0]), y = TM_read(stm, tx, a[1]);
                    TM_write(stm, tx, a[0], x - 1);
                    TM_write(stm, tx, a[1], y + 1);
                });
                ++done;
            }
            return done;
        };
        RoundReport rep = eng.runRoundBatches(HETM_KERNEL_BANK, sizeof(hetm_bank_tx), recording, worker);
        record();  // the last launched batch (the engine may stop without polling again)
        batches += rep.dev_batches;
        executed += rep.dev_committed;
        if (rep.conflict || rep.dev_batches != round_tx.size() / B) {
            std::printf("round %d: conflict=%d batches=%u recorded=%zu\n", r, (int)rep.conflict, rep.dev_batches,
                        round_tx.size() / B);
            ok = false;
        }
        const auto& hl = eng.lastRoundLog();
        orc_apply_log_ts_order(ref.data(), 0, reinterpret_cast<const orc_entry*>(hl.data()), hl.size());
        std::vector<uint64_t> order(round_tk.size());
        const uint64_t m = orc_order_by_ticket(round_tk.data(), round_tk.size(), order.data());
        orc_bank_replay(ref.data(), 0, round_tx.data(), order.data(), m, nullptr, nullptr, nullptr, 1024, 16384);
        std::vector<uint64_t> dv(W);
        check_rc(hetm_dev_download(dev, HETM_REPLICA_DEV, 0, dv.data(), W), "download");
        if (std::memcmp(ref.data(), host, W * 8) || std::memcmp(dv.data(), host, W * 8)) {
            std::printf("round %d: replicas differ from the oracle replay\n", r);
            ok = false;
        }
    }
    // drain: whatever the queue still holds is exactly the unexecuted tail
    if (executed + q.size() != submitted) {
        std::printf("exactly-once violated: executed %llu + queued %llu != submitted %llu\n",
                    (unsigned long long)executed, (unsigned long long)q.size(), (unsigned long long)submitted);
        ok = false;
    }
    std::printf("{\"rounds\": %d, \"batch\": %llu, \"batches\": %llu, \"submitted\": %llu, \"executed\": %llu, "
                "\"queued_tail\": %llu, \"ok\": %d}\n",
                rounds, (unsigned long long)B, (unsigned long long)batches, (unsigned long long)submitted,
                (unsigned long long)executed, (unsigned long long)q.size(), (int)ok);
    hetm_host_free(host);
    hetm_dev_close(dev);
    return ok ? 0 : 1;
}
