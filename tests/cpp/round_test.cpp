// round_test.cpp — end-to-end SHeTM rounds with a LIVE host producer:
// host worker threads run bank transfers through the host TL2 STM
// (include/hetm_b200/host_tm.hpp) while the GPU runs a bank batch; the
// engine (include/hetm_b200/engine.hpp) streams the host write log with
// early validation, validates, and merges (FavorHost).  TEST INFRASTRUCTURE:
// every round is checked against the CPU oracle (oracle/liboracle.so):
//   committed round: S' = bank_replay(apply_log_ts_order(S, host log), device
//                    batch in ticket order)
//   aborted round:   S' = apply_log_ts_order(S, host log)
// plus host replica == device replica and the bank sum.
//
//   round_test [rounds] [log2 words] [batch] [host threads] [conflict every k]
// Exit 0 = all rounds bit-exact; prints one JSON line with the totals.
#include <atomic>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "hetm_b200/capi.h"
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
    const int rounds = argc > 1 ? std::atoi(argv[1]) : 6;
    const int log2w = argc > 2 ? std::atoi(argv[2]) : 20;
    const uint64_t B = argc > 3 ? std::strtoull(argv[3], nullptr, 10) : (1u << 14);
    const int T = argc > 4 ? std::atoi(argv[4]) : 4;
    const int conflict_every = argc > 5 ? std::atoi(argv[5]) : 3;
    const uint64_t W = 1ull << log2w, half = W / 2;

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
    check_rc(hetm_dev_upload(dev, HETM_REPLICA_DEV, 0, host, W), "upload");
    check_rc(hetm_dev_merge_commit(dev, host, nullptr), "merge");
    check_rc(hetm_dev_merge_wait(dev), "merge_wait");
    check_rc(hetm_dev_clear_round(dev, 0), "clear");

    HostStm stm(host, W, 20);
    WriteLog log(T);
    stm.setCommitCallback([&](int t, std::span<const hetm_log_entry> es) { log.append(t, es); });
    EngineConfig ec;
    ec.chunk_entries = 1u << 12;
    ec.keep_round_log = true;
    Engine eng(dev, stm, log, host, ec);

    std::vector<uint64_t> ref(host, host + W), dev_words(W), tickets(B), order(B);
    std::vector<orc_bank_tx> txs(B);
    uint64_t host_total = 0, dev_total = 0, n_conflict = 0, n_cut = 0;
    bool ok = true;
    for (int r = 0; r < rounds && ok; ++r) {
        const bool steal = conflict_every > 0 && r % conflict_every == conflict_every - 1;
        orc_gen_bank_batch(1000 + r, B, 0, half, txs.data());  // device partition [0, W/2)
        const uint64_t per_thread = 1500;
        auto worker = [&](int t, const std::atomic<bool>& stop) -> uint64_t {
            uint64_t s = orc_splitmix64(7919u * r + t + 1), done = 0;
            for (uint64_t k = 0; k < per_thread && !stop.load(std::memory_order_relaxed); ++k) {
                uint64_t a[4];
                for (int j = 0; j < 4; ++j) {
                    s = orc_splitmix64(s);
                    // host partition [W/2, W); a stealing round also WRITES into the device half
                    a[j] = (steal && j == 0) ? (s % half) : half + s % half;
                }
                if (a[0] == a[1]) continue;
                s = orc_splitmix64(s);
                const uint64_t amt = s % 100 + 1;
                stm.atomically(t, [&](HostStm::Tx& tx) {
                    const uint64_t x = TM_read(stm, tx, a[0]);
                    const uint64_t y = TM_read(stm, tx, a[1]);
                    (void)TM_read(stm, tx, a[2]);
                    (void)TM_read(stm, tx, a[3]);
                    TM_write(stm, tx, a[0], x - amt);
                    TM_write(stm, tx, a[1], y + amt);
                });
                ++done;
            }
            return done;
        };
        RoundReport rep = eng.runRound(HETM_KERNEL_BANK, txs.data(), sizeof(hetm_bank_tx), B, tickets.data(), worker);
        host_total += rep.host_commits;
        n_conflict += rep.conflict;
        n_cut += rep.cut_short;
        if (steal != rep.conflict) {
            std::printf("round %d: conflict=%d but steal=%d\n", r, (int)rep.conflict, (int)steal);
            ok = false;
        }
        std::printf("{\"round\": %d, \"conflict\": %d, \"cut_short\": %d, \"host_commits\": %llu, \"dev_committed\": %llu, "
                    "\"log_entries\": %llu, \"chunks\": %llu, \"exec_ms\": %.3f, \"validate_ms\": %.3f, \"merge_ms\": %.3f}\n",
                    r, (int)rep.conflict, (int)rep.cut_short, (unsigned long long)rep.host_commits,
                    (unsigned long long)rep.dev_committed, (unsigned long long)rep.log_entries,
                    (unsigned long long)rep.chunks, rep.exec_ms, rep.validate_ms, rep.merge_ms);
        if (!rep.conflict) dev_total += rep.dev_committed;
        // exact oracle replay of the round
        const auto& hl = eng.lastRoundLog();
        orc_apply_log_ts_order(ref.data(), 0, reinterpret_cast<const orc_entry*>(hl.data()), hl.size());
        if (!rep.conflict) {
            const uint64_t m = orc_order_by_ticket(tickets.data(), B, order.data());
            orc_bank_replay(ref.data(), 0, txs.data(), order.data(), m, nullptr, nullptr, nullptr, 1024, 16384);
        }
        if (std::memcmp(ref.data(), host, W * 8) != 0) {
            std::printf("round %d: host replica != oracle replay\n", r);
            ok = false;
        }
        check_rc(hetm_dev_download(dev, HETM_REPLICA_DEV, 0, dev_words.data(), W), "download");
        if (std::memcmp(dev_words.data(), host, W * 8) != 0) {
            std::printf("round %d: device replica != host replica\n", r);
            ok = false;
        }
        uint64_t sum = 0;
        for (uint64_t i = 0; i < W; ++i) sum += host[i];
        if (sum != 1000 * W) {
            std::printf("round %d: bank sum broken\n", r);
            ok = false;
        }
    }
    std::printf("{\"rounds\": %d, \"ok\": %d, \"host_commits\": %llu, \"dev_commits\": %llu, \"conflict_rounds\": %llu, "
                "\"cut_short\": %llu, \"host_aborts\": %llu}\n",
                rounds, (int)ok, (unsigned long long)host_total, (unsigned long long)dev_total,
                (unsigned long long)n_conflict, (unsigned long long)n_cut, (unsigned long long)stm.aborts());
    hetm_host_free(host);
    hetm_dev_close(dev);
    return ok ? 0 : 1;
}
