// live_round.cpp — end-to-end SHeTM rounds with a LIVE host producer at
// BASELINE configs[1] scale: the bench runner of the
// reference's round loop (engine.runRound), over this
// library only — no oracle, no checks beyond the bank-sum invariant.
//
// Per round (include/hetm_b200/engine.hpp): the GPU-controller thread runs one
// 2^20-transaction bank batch on the device half [0, W/2) from a pinned host
// buffer while T host workers commit bank transfers through the TL2 host TM
// (host_tm.hpp) on the host half [W/2, W); the engine streams the host write
// log in chunks (early validation every ev_period chunks), keeps the host
// committing after the execution phase until at most cutoff_chunks chunks
// are undelivered (hostCutoff), validates + applies the
// tail, reads the verdict and merges (delta merge staged right after the
// execution phase).  Partitioned accesses: no conflicts, every round commits.
//
//   hetm_live_round [rounds] [log2 words] [batch] [host threads] [cutoff chunks] [ev period] [chunk entries]
//                   [pipeline merge 1|0: a committed round's merge lands under the next round's device
//                    batches, EngineConfig::pipeline_merge; default 1]
//
// Prints one JSON line: committed host + device transactions per second of
// wall clock over the timed rounds (the first round is warm-up).
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <thread>
#include <vector>

#include "hetm_b200/capi.h"
#include "hetm_b200/engine.hpp"
#include "hetm_b200/host_tm.hpp"

using namespace hetm::b200;

static uint64_t mix(uint64_t x) {  // splitmix64 finalizer: host-side address draws
    x += 0x9e3779b97f4a7c15ull;
    x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
    x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
    return x ^ (x >> 31);
}

int main(int argc, char** argv) {
    const int rounds = argc > 1 ? std::atoi(argv[1]) : 12;
    const int log2w = argc > 2 ? std::atoi(argv[2]) : 27;
    const uint64_t B = argc > 3 ? std::strtoull(argv[3], nullptr, 10) : (1u << 20);
    int T = argc > 4 ? std::atoi(argv[4]) : 0;
    const uint32_t cutoff = argc > 5 ? (uint32_t)std::atoi(argv[5]) : 4;
    const uint32_t ev_period = argc > 6 ? (uint32_t)std::atoi(argv[6]) : 8;
    const uint64_t chunk = argc > 7 ? std::strtoull(argv[7], nullptr, 10) : (1u << 16);
    const bool pipeline = argc > 8 ? std::atoi(argv[8]) != 0 : true;  // merge lands under the next batch
    if (T <= 0) {  // every core but the controller's and the GPU-controller thread's
        const int hw = (int)std::thread::hardware_concurrency();
        T = hw > 3 ? hw - 2 : 1;
    }
    const uint64_t W = 1ull << log2w, half = W / 2;

    hetm_dev_config cfg;
    hetm_dev_config_default(&cfg);
    cfg.size_words = W;
    cfg.rs_gran_bytes = 1024;
    cfg.flags = HETM_CFG_MERGE_DELTA;
    hetm_dev* dev = nullptr;
    int rc = hetm_dev_open(&cfg, &dev);
    if (rc != HETM_OK) {
        std::printf("{\"error\": \"open: %s\"}\n", hetm_strerror(rc));
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

    // two pinned device batches, alternating (generated before the rounds)
    hetm_bank_tx* txs[2];
    uint64_t* tickets = nullptr;
    for (int k = 0; k < 2; ++k) {
        check_rc(hetm_host_alloc(B * sizeof(hetm_bank_tx), reinterpret_cast<void**>(&txs[k])), "host_alloc");
        check_rc(hetm_gen_bank_batch(1000 + k, B, 0, half, txs[k]), "gen");
    }
    check_rc(hetm_host_alloc(B * 8, reinterpret_cast<void**>(&tickets)), "host_alloc");

    HostStm stm(host, W, 24);
    WriteLog log(T);
    stm.setCommitCallback([&](int t, std::span<const hetm_log_entry> es) { log.append(t, es); });
    EngineConfig ec;
    ec.chunk_entries = chunk;
    ec.cutoff_chunks = cutoff;
    ec.pipeline_merge = pipeline;
    ec.ev_period = ev_period;
    Engine eng(dev, stm, log, host, ec);

    uint64_t host_commits = 0, dev_commits = 0, log_entries = 0, chunks = 0, cut_chunks = 0, commits = 0;
    double exec_ms = 0, val_ms = 0, merge_ms = 0, blocked_ms = 0;
    std::chrono::steady_clock::time_point t0{};
    for (int r = 0; r <= rounds; ++r) {
        if (r == 1) {  // round 0 is warm-up
            t0 = std::chrono::steady_clock::now();
            host_commits = dev_commits = log_entries = chunks = cut_chunks = commits = 0;
            exec_ms = val_ms = merge_ms = blocked_ms = 0;
        }
        auto worker = [&, r](int t, const RoundContext& ctx) -> uint64_t {
            uint64_t s = mix(7919u * (uint64_t)r + (uint64_t)t + 1), done = 0;
            while (!ctx.stop.load(std::memory_order_relaxed)) {
                uint64_t a[4];
                for (int j = 0; j < 4; ++j) a[j] = half + (s = mix(s)) % half;
                if (a[0] == a[1]) continue;
                const uint64_t amt = (s = mix(s)) % 100 + 1;
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
        RoundReport rep = eng.runRoundBatches(HETM_KERNEL_BANK, sizeof(hetm_bank_tx), [&](uint32_t k, Engine::Batch& b) {
            if (k >= 1) return false;
            b = Engine::Batch{txs[r & 1], B, tickets};
            return true;
        }, worker);
        if (rep.outcome == Outcome::Commit) ++commits;
        if (rep.outcome != Outcome::HostAborted) host_commits += rep.host_commits;
        if (rep.outcome != Outcome::DeviceAborted) dev_commits += rep.dev_committed;
        log_entries += rep.log_entries;
        chunks += rep.chunks;
        cut_chunks += rep.cutoff_chunks;
        exec_ms += rep.exec_ms;
        val_ms += rep.validate_ms;
        merge_ms += rep.merge_ms;
        blocked_ms += rep.host_blocked_ms;
    }
    eng.drain();  // the last round's merge lands inside the timed region
    const double wall = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    uint64_t sum = 0;
    for (uint64_t i = 0; i < W; ++i) sum += host[i];
    const bool sum_ok = sum == 1000 * W;
    std::printf("{\"rounds\": %d, \"committed_rounds\": %llu, \"host_threads\": %d, \"stmr_words\": %llu, "
                "\"batch_tx\": %llu, \"cutoff_chunks\": %u, \"ev_period\": %u, \"chunk_entries\": %llu, "
                "\"wall_s\": %.6f, \"tx_per_s\": %.1f, \"dev_tx_per_s\": %.1f, \"host_tx_per_s\": %.1f, "
                "\"host_commits\": %llu, \"dev_commits\": %llu, \"log_entries_per_round\": %.1f, "
                "\"chunks_per_round\": %.2f, \"chunks_after_exec_per_round\": %.2f, \"exec_ms\": %.4f, "
                "\"validate_ms\": %.4f, \"merge_ms\": %.4f, \"host_blocked_ms\": %.4f, "
                "\"staging_buffers\": %zu, \"host_aborts\": %llu, \"pipeline_merge\": %s, \"bank_sum_ok\": %s}\n",
                rounds, (unsigned long long)commits, T, (unsigned long long)W, (unsigned long long)B, cutoff,
                ev_period, (unsigned long long)chunk, wall, (double)(host_commits + dev_commits) / wall,
                (double)dev_commits / wall, (double)host_commits / wall, (unsigned long long)host_commits,
                (unsigned long long)dev_commits, (double)log_entries / rounds, (double)chunks / rounds,
                (double)cut_chunks / rounds, exec_ms / rounds, val_ms / rounds, merge_ms / rounds,
                blocked_ms / rounds, eng.stagingBuffers(), (unsigned long long)stm.aborts(),
                pipeline ? "true" : "false", sum_ok ? "true" : "false");
    for (auto* p : txs) hetm_host_free(p);
    hetm_host_free(tickets);
    hetm_host_free(host);
    hetm_dev_close(dev);
    return sum_ok ? 0 : 1;
}
