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
//   round_test [rounds] [log2 words] [batch] [host threads] [conflict every k] [host|device] [starvation k]
//              [batches per round] [early validation 1|0] [cutoff chunks] [bus delay us/unit]
//              [host tx per thread per round (0: until the cut-off)] [early-validation period k]
//              [pipelined merge 1|0]
// policy host (FavorHost, default) or device (FavorDevice: a conflicting round
// is HostAborted, S' = device batch replay on S, host effects discarded).
// conflict every k = 1 makes every round conflict (starvation-guard test).
// Exit 0 = all rounds bit-exact; prints one JSON line per round + the totals.
#include <algorithm>
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
    const bool favor_device = argc > 6 && std::strcmp(argv[6], "device") == 0;
    const uint32_t starvation_k = argc > 7 ? (uint32_t)std::atoi(argv[7]) : 3;
    const uint32_t n_batches = argc > 8 ? (uint32_t)std::atoi(argv[8]) : 1;
    const bool early = argc > 9 ? std::atoi(argv[9]) != 0 : true;
    const uint32_t cutoff = argc > 10 ? (uint32_t)std::atoi(argv[10]) : 4;
    const double bus_delay = argc > 11 ? std::atof(argv[11]) : 0.0;
    const uint64_t per_thread_arg = argc > 12 ? std::strtoull(argv[12], nullptr, 10) : 1500;
    const uint32_t ev_period = argc > 13 ? (uint32_t)std::atoi(argv[13]) : 8;
    const bool pipeline = argc > 14 && std::atoi(argv[14]) != 0;  // EngineConfig::pipeline_merge (+ drain() per check)
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
    ec.chunk_entries = n_batches > 1 ? 256 : (1u << 12);  // small chunks: early validation during execution
    ec.early_validation = early;
    ec.keep_round_log = true;
    ec.policy = favor_device ? Policy::FavorDevice : Policy::FavorHost;
    ec.starvation_k = starvation_k;
    ec.cutoff_chunks = cutoff;
    ec.bus_real_delay_us_per_unit = bus_delay;
    ec.ev_period = ev_period;
    ec.pipeline_merge = pipeline;
    Engine eng(dev, stm, log, host, ec);
    double blocked_ms = 0;
    uint64_t cutoff_chunks = 0, log_total = 0;

    std::vector<uint64_t> ref(host, host + W), dev_words(W), tickets((uint64_t)B * n_batches), order((uint64_t)B * n_batches);
    std::vector<orc_bank_tx> txs((uint64_t)B * n_batches);
    uint64_t batches_total = 0, wasted = 0;
    uint64_t host_total = 0, dev_total = 0, n_conflict = 0, n_cut = 0, n_guard = 0;
    uint32_t run_aborts = 0, max_run_aborts = 0;
    bool ok = true;
    std::vector<uint64_t> start(W);
    for (int r = 0; r < rounds && ok; ++r) {
        const bool steal = conflict_every > 0 && r % conflict_every == conflict_every - 1;
        for (uint32_t k = 0; k < n_batches; ++k)  // device partition [0, W/2)
            orc_gen_bank_batch(1000 + 64 * r + k, B, 0, half, txs.data() + (uint64_t)k * B);
        std::fill(tickets.begin(), tickets.end(), ~0ull);
        const uint64_t per_thread = per_thread_arg ? per_thread_arg : ~0ull;
        auto worker = [&](int t, const RoundContext& ctx) -> uint64_t {
            uint64_t s = orc_splitmix64(7919u * r + t + 1), done = 0;
            for (uint64_t k = 0; k < per_thread && !ctx.stop.load(std::memory_order_relaxed); ++k) {
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
                    if (!ctx.updates_allowed) return;  // starvation guard: read-only transaction
                    TM_write(stm, tx, a[0], x - amt);
                    TM_write(stm, tx, a[1], y + amt);
                });
                ++done;
            }
            return done;
        };
        RoundReport rep = eng.runRoundBatches(HETM_KERNEL_BANK, sizeof(hetm_bank_tx), [&](uint32_t k, Engine::Batch& b) {
            if (k >= n_batches) return false;
            b = Engine::Batch{txs.data() + (uint64_t)k * B, B, tickets.data() + (uint64_t)k * B};
            return true;
        }, worker);
        eng.drain();  // pipeline_merge: the round's merge lands before the host replica is read below
        batches_total += rep.dev_batches;
        blocked_ms += rep.host_blocked_ms;
        cutoff_chunks += rep.cutoff_chunks;
        log_total += rep.log_entries;
        if (rep.outcome == Outcome::DeviceAborted) wasted += rep.dev_committed;
        n_conflict += rep.conflict;
        n_cut += rep.cut_short;
        n_guard += !rep.updates_allowed;
        const bool host_updates = steal && rep.updates_allowed;
        if (host_updates != rep.conflict) {
            std::printf("round %d: conflict=%d but steal=%d updates=%d\n", r, (int)rep.conflict, (int)steal,
                        (int)rep.updates_allowed);
            ok = false;
        }
        std::printf("%s\n", rep.json().c_str());
        if (rep.outcome != Outcome::HostAborted) host_total += rep.host_commits;
        if (rep.outcome != Outcome::DeviceAborted) dev_total += rep.dev_committed;
        run_aborts = rep.outcome == Outcome::DeviceAborted ? run_aborts + 1 : 0;
        max_run_aborts = std::max(max_run_aborts, run_aborts);
        // exact oracle replay of the round
        const auto& hl = eng.lastRoundLog();
        if (rep.outcome != Outcome::HostAborted)
            orc_apply_log_ts_order(ref.data(), 0, reinterpret_cast<const orc_entry*>(hl.data()), hl.size());
        if (rep.outcome != Outcome::DeviceAborted) {
            const uint64_t m = orc_order_by_ticket(tickets.data(), tickets.size(), order.data());
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
    if (!favor_device && max_run_aborts > starvation_k) {  // device commits within K+1 rounds
        std::printf("starvation guard failed: %u consecutive device aborts\n", max_run_aborts);
        ok = false;
    }
    std::printf("{\"rounds\": %d, \"ok\": %d, \"policy\": \"%s\", \"host_commits\": %llu, \"dev_commits\": %llu, "
                "\"conflict_rounds\": %llu, \"cut_short\": %llu, \"guard_rounds\": %llu, \"max_consecutive_device_aborts\": %u, "
                "\"host_aborts\": %llu, \"device_batches\": %llu, \"wasted_device_tx\": %llu, "
                "\"host_blocked_ms\": %.3f, \"cutoff_chunks\": %llu, \"log_entries\": %llu, \"staging_buffers\": %zu}\n",
                rounds, (int)ok, favor_device ? "FavorDevice" : "FavorHost", (unsigned long long)host_total,
                (unsigned long long)dev_total, (unsigned long long)n_conflict, (unsigned long long)n_cut,
                (unsigned long long)n_guard, max_run_aborts, (unsigned long long)stm.aborts(),
                (unsigned long long)batches_total, (unsigned long long)wasted, blocked_ms,
                (unsigned long long)cutoff_chunks, (unsigned long long)log_total, eng.stagingBuffers());
    hetm_host_free(host);
    hetm_dev_close(dev);
    return ok ? 0 : 1;
}
