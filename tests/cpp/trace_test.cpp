// trace_test.cpp — checker traces of LIVE engine rounds:
// host workers run bank transfers through HostStm while the GPU runs bank
// batches; the engine records every event (Engine::setTrace) and the CPU
// checker (oracle/checker.c, TEST INFRASTRUCTURE) verifies P1 over the
// finally committed transactions and P2-dagger over the speculative ones.
// The partitions swap every round (device [0, W/2) and host [W/2, W) on even
// rounds, the reverse on odd ones), so every round reads what the other side
// wrote in the previous one; every 3rd round the host also writes into the
// device half (a conflict: DeviceAborted under FavorHost).
//
//   trace_test [rounds] [device faults HETM_FAULT_*] [engine faults ENGINE_FAULT_*] [dump path] [host|device]
// (policy: FavorHost, or FavorDevice — conflicting rounds are then HostAborted
// and P2-dagger checks the host's speculative set)
// Exit 0 iff the verdicts are as expected: both checks pass with no fault, and
// at least one fails (the mutation is caught) with any fault.  One JSON line.
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "hetm_b200/capi.h"
#include "hetm_b200/engine.hpp"
#include "hetm_b200/host_tm.hpp"
#include "hetm_b200/trace.hpp"

extern "C" {  // oracle/hetm_oracle.h (test infrastructure)
typedef struct { uint32_t acct[4]; uint64_t amount; } orc_bank_tx;
void orc_gen_bank_batch(uint64_t seed, uint64_t n, uint64_t lo, uint64_t span, orc_bank_tx* out);
uint64_t orc_splitmix64(uint64_t x);
typedef struct {
    int verdict, reason;
    uint64_t tx, addr, expected, got;
    uint32_t round;
    uint64_t checked_txs, checked_reads;
} orc_check_result;
int orc_check_p1(const void* ev, uint64_t n, const uint64_t* init, uint64_t words, orc_check_result* res);
int orc_check_p2dagger(const void* ev, uint64_t n, const uint64_t* init, uint64_t words, orc_check_result* res);
}

using namespace hetm::b200;

int main(int argc, char** argv) {
    const int rounds = argc > 1 ? std::atoi(argv[1]) : 9;
    const uint32_t dev_fault = argc > 2 ? (uint32_t)std::strtoul(argv[2], nullptr, 0) : 0;
    const uint32_t eng_fault = argc > 3 ? (uint32_t)std::strtoul(argv[3], nullptr, 0) : 0;
    const std::string dump = argc > 4 ? argv[4] : "";
    const bool favor_device = argc > 5 && std::strcmp(argv[5], "device") == 0;
    const uint64_t W = 1ull << 18, half = W / 2, B = 1u << 12;
    const int T = 4;

    hetm_dev_config cfg;
    hetm_dev_config_default(&cfg);
    cfg.size_words = W;
    cfg.rs_gran_bytes = 1024;
    cfg.flags = HETM_CFG_MERGE_DELTA;
    hetm_dev* dev = nullptr;
    int rc = hetm_dev_open(&cfg, &dev);
    if (rc != HETM_OK) {
        std::printf("open: %s\n", hetm_strerror(rc));
        return rc == HETM_ERR_NO_DEVICE ? 3 : 1;
    }
    check_rc(hetm_dev_register_kernel(dev, HETM_KERNEL_BANK), "register");
    uint64_t* host = nullptr;
    check_rc(hetm_host_alloc(W * 8, reinterpret_cast<void**>(&host)), "host_alloc");
    for (uint64_t i = 0; i < W; ++i) host[i] = 1000;
    const std::vector<uint64_t> init(host, host + W);
    check_rc(hetm_dev_upload(dev, HETM_REPLICA_DEV, 0, host, W), "upload");
    check_rc(hetm_dev_merge_commit(dev, host, nullptr), "merge");
    check_rc(hetm_dev_merge_wait(dev), "merge_wait");
    check_rc(hetm_dev_clear_round(dev, 0), "clear");
    check_rc(hetm_dev_set_fault(dev, dev_fault), "set_fault");

    HostStm stm(host, W, 18);
    WriteLog log(T);
    stm.setCommitCallback([&](int t, std::span<const hetm_log_entry> es) { log.append(t, es); });
    EngineConfig ec;
    ec.chunk_entries = 256;
    ec.fault = eng_fault;
    ec.policy = favor_device ? Policy::FavorDevice : Policy::FavorHost;
    Engine eng(dev, stm, log, host, ec);
    Trace trace(W, "{\"kernel\": \"bank\", \"batch\": " + std::to_string(B) + ", \"host_threads\": " +
                       std::to_string(T) + ", \"dev_fault\": " + std::to_string(dev_fault) +
                       ", \"engine_fault\": " + std::to_string(eng_fault) + "}");
    eng.setTrace(&trace);

    std::vector<orc_bank_tx> txs(B);
    std::vector<uint64_t> tickets(B);
    int n_conflict = 0;
    for (int r = 0; r < rounds; ++r) {
        const uint64_t dev_lo = (r % 2) ? half : 0, host_lo = (r % 2) ? 0 : half;
        const bool steal = r % 3 == 2;
        orc_gen_bank_batch(5000 + r, B, dev_lo, half, txs.data());
        auto worker = [&](int t, const RoundContext& ctx) -> uint64_t {
            uint64_t s = orc_splitmix64(7919u * r + t + 1), done = 0;
            for (int k = 0; k < 600 && !ctx.stop.load(std::memory_order_relaxed); ++k) {
                uint64_t a[4];
                for (int j = 0; j < 4; ++j) {
                    s = orc_splitmix64(s);
                    a[j] = (steal && j == 0) ? dev_lo + s % half : host_lo + s % half;
                }
                if (a[0] == a[1]) continue;
                s = orc_splitmix64(s);
                const uint64_t amt = s % 100 + 1;
                stm.atomically(t, [&](HostStm::Tx& tx) {
                    const uint64_t x = TM_read(stm, tx, a[0]);
                    const uint64_t y = TM_read(stm, tx, a[1]);
                    (void)TM_read(stm, tx, a[2]);
                    (void)TM_read(stm, tx, a[3]);
                    if (!ctx.updates_allowed) return;
                    TM_write(stm, tx, a[0], x - amt);
                    TM_write(stm, tx, a[1], y + amt);
                });
                ++done;
            }
            return done;
        };
        RoundReport rep = eng.runRound(HETM_KERNEL_BANK, txs.data(), sizeof(hetm_bank_tx), B, tickets.data(), worker);
        n_conflict += rep.conflict;
    }
    const auto ev = trace.events();
    if (!dump.empty()) trace.dump(dump);
    orc_check_result p1{}, p2{};
    orc_check_p1(ev.data(), ev.size(), init.data(), W, &p1);
    orc_check_p2dagger(ev.data(), ev.size(), init.data(), W, &p2);
    const bool faulty = dev_fault || eng_fault;
    const bool caught = p1.verdict != 0 || p2.verdict != 0;
    const bool ok = faulty ? caught : (p1.verdict == 0 && p2.verdict == 0);
    std::printf("{\"rounds\": %d, \"policy\": \"%s\", \"dev_fault\": %u, \"engine_fault\": %u, \"events\": %zu, \"conflict_rounds\": %d, "
                "\"p1\": {\"verdict\": %d, \"reason\": %d, \"tx\": %llu, \"addr\": %llu, \"expected\": %llu, "
                "\"got\": %llu, \"round\": %u, \"txs\": %llu, \"reads\": %llu}, "
                "\"p2dagger\": {\"verdict\": %d, \"reason\": %d, \"round\": %u, \"txs\": %llu, \"reads\": %llu}, "
                "\"ok\": %d}\n",
                rounds, favor_device ? "FavorDevice" : "FavorHost", dev_fault, eng_fault, ev.size(), n_conflict, p1.verdict, p1.reason,
                (unsigned long long)p1.tx, (unsigned long long)p1.addr, (unsigned long long)p1.expected,
                (unsigned long long)p1.got, p1.round, (unsigned long long)p1.checked_txs,
                (unsigned long long)p1.checked_reads, p2.verdict, p2.reason, p2.round,
                (unsigned long long)p2.checked_txs, (unsigned long long)p2.checked_reads, (int)ok);
    hetm_host_free(host);
    hetm_dev_close(dev);
    return ok ? 0 : 1;
}
