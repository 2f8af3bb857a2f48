// Compiles include/hetm_b200/hetm_gpu.hpp and host_tm.hpp against the
// REFERENCE headers and exercises them as a reference maintainer would:
//   1. a reference-typed host worker loop — transactions through the host TM,
//      `catch (hetm::TxAbort&)` retries, `hetm::OutOfBoundsError` on a bad
//      address, commits appended to the reference's own hetm::WriteLog;
//   2. on the GPU, that log streamed through a 2-buffer pinned staging ring
//      whose buffers are recycled as soon as their chunk is delivered
//      (hetm_dev_stream_chunk_ex handles, bus.hpp:51-56 Delivery) — before
//      the round's verdict — then verdict + mergeCommit, replicas compared.
// Without a GPU the device open must throw (no CPU fallback): exit 3.
#include <atomic>
#include <cstdio>
#include <cstring>
#include <thread>
#include <vector>

#include "hetm_b200/hetm_gpu.hpp"
#include "hetm_b200/host_tm.hpp"

#ifndef HETM_B200_REFERENCE_TYPES
#error "binding_smoke must be compiled against the reference headers (-I <reference>/proj/include)"
#endif
static_assert(std::is_same_v<hetm::b200::TxAbort, hetm::TxAbort>, "host TM aborts are the reference's TxAbort");
static_assert(std::is_same_v<hetm::b200::OutOfBoundsError, hetm::OutOfBoundsError>);

namespace {
constexpr std::size_t kWords = 1 << 12;      // STMR words; the host owns [2048, 4096)
constexpr std::size_t kChunk = 64;           // entries per streamed chunk
constexpr int kThreads = 2, kTxPerThread = 2000;

// Reference-typed worker loop over the host TM: transfers between 8 hot
// accounts of the host half, retried on hetm::TxAbort.
std::size_t run_host_workers(hetm::b200::HostStm& stm, std::atomic<std::size_t>& aborts) {
    std::vector<std::thread> ws;
    for (int t = 0; t < kThreads; ++t)
        ws.emplace_back([&, t] {
            hetm::b200::HostStm::Tx tx;
            for (int i = 0; i < kTxPerThread; ++i) {
                const hetm::WordIdx a = 2048 + (i * 3 + t) % 8, b = 2048 + (i * 5 + 1 + t) % 8;
                for (;;) {
                    try {
                        hetm::b200::TM_begin(stm, tx, t);
                        const hetm::Word va = hetm::b200::TM_read(stm, tx, a);
                        const hetm::Word vb = hetm::b200::TM_read(stm, tx, b);
                        hetm::b200::TM_write(stm, tx, a, va - 1);
                        hetm::b200::TM_write(stm, tx, b, vb + 1);
                        hetm::b200::TM_commit(stm, tx);
                        break;
                    } catch (hetm::TxAbort&) {  // the reference's abort type: retry
                        aborts.fetch_add(1, std::memory_order_relaxed);
                    }
                }
            }
        });
    for (auto& w : ws) w.join();
    return static_cast<std::size_t>(kThreads) * kTxPerThread;
}
}  // namespace

int main() {
    // ---- 1. host TM on the reference types (CPU only)
    std::vector<hetm::Word> host(kWords, 1000);
    hetm::WriteLog refLog;  // the reference's WriteLog (write_log.hpp:31)
    for (int t = 0; t < kThreads; ++t) refLog.registerThread();
    hetm::b200::HostStm stm(host.data(), host.size(), 12);
    stm.setCommitCallback(hetm::b200::commitTo(refLog));
    std::atomic<std::size_t> aborts{0};
    {  // a forced conflict: tx1 read word 2100, tx2 commits it, tx1's next read must abort
        hetm::b200::HostStm::Tx tx1, tx2;
        hetm::b200::TM_begin(stm, tx1, 0);
        (void)hetm::b200::TM_read(stm, tx1, 2100);
        hetm::b200::TM_begin(stm, tx2, 1);
        hetm::b200::TM_write(stm, tx2, 2100, hetm::b200::TM_read(stm, tx2, 2100) + 0);
        hetm::b200::TM_commit(stm, tx2);
        try {
            hetm::b200::TM_write(stm, tx1, 2100, 5);
            hetm::b200::TM_commit(stm, tx1);
        } catch (hetm::TxAbort&) {
            aborts.fetch_add(1);
        }
        if (aborts.load() != 1) return 2;
    }
    const std::size_t workers = run_host_workers(stm, aborts), committed = workers + 1;
    bool oob = false;
    try {
        hetm::b200::HostStm::Tx tx;
        hetm::b200::TM_begin(stm, tx, 0);
        (void)hetm::b200::TM_read(stm, tx, kWords + 5);
    } catch (const hetm::OutOfBoundsError&) {
        oob = true;
    }
    hetm::Word sum = 0;
    for (std::size_t a = 2048; a < 2056; ++a) sum += host[a];
    const std::size_t logged = refLog.totalEntries();
    std::printf("host worker loop ok: %zu tx committed, %zu TxAbort retries, %zu log entries, oob=%d, sum_ok=%d\n",
                committed, aborts.load(), logged, (int)oob, (int)(sum == 8 * 1000));
    if (!oob || logged != 2 * workers + 1 || sum != 8 * 1000) return 1;

    try {
        // ---- 2. device round fed by a 2-buffer pinned staging ring
        hetm::b200::GpuDevice dev(kWords, 64);
        dev.registerKernel(HETM_KERNEL_BANK);
        std::vector<hetm::Word> init(kWords, 1000);
        for (std::size_t a = 0; a < kWords; ++a) dev.rawWrite(hetm::Replica::Dev, a, init[a]);
        std::vector<hetm_bank_tx> txs(256);
        for (std::size_t i = 0; i < txs.size(); ++i) {  // the device half [0, 2048)
            txs[i].acct[0] = i % 2048;
            txs[i].acct[1] = (i * 7 + 1) % 2048;
            txs[i].acct[2] = (i * 13 + 2) % 2048;
            txs[i].acct[3] = (i * 31 + 3) % 2048;
            txs[i].amount = 1;
        }
        auto tickets = dev.executeBatch(HETM_KERNEL_BANK, txs.data(), sizeof(hetm_bank_tx), txs.size());
        void* ring[2] = {nullptr, nullptr};
        for (auto& r : ring) hetm::b200::check(hetm_host_alloc(kChunk * sizeof(hetm_log_entry), &r));
        std::uint64_t handle[2] = {0, 0};
        bool busy[2] = {false, false};
        std::size_t chunks = 0, recycled = 0;
        std::uint64_t seq = 0;
        for (int t = 0; t < refLog.threadCount(); ++t) {
            for (std::size_t from = 0; from < refLog.entryCount(t); from += kChunk) {
                const int b = static_cast<int>(chunks % 2);
                if (busy[b]) {  // recycle: wait for THIS buffer's delivery, not for the verdict
                    dev.waitDelivered(handle[b]);
                    if (!dev.delivered(handle[b])) return 4;
                    ++recycled;
                }
                const auto part = refLog.slice(t, from, kChunk);
                std::memcpy(ring[b], part.data(), part.size() * sizeof(hetm_log_entry));
                hetm_delivery dl{};
                hetm::b200::check(hetm_dev_stream_chunk_ex(dev.handle(), static_cast<hetm_log_entry*>(ring[b]),
                                                           part.size(), t, seq++, HETM_APPLY, &dl));
                handle[b] = dl.handle;
                busy[b] = true;
                ++chunks;
            }
        }
        const bool conflict = dev.roundVerdict();
        dev.mergeCommit(host);
        dev.mergeWait();
        for (auto& r : ring) hetm_host_free(r);
        bool match = true;
        for (std::size_t a = 0; a < kWords; ++a) match = match && host[a] == dev.rawRead(hetm::Replica::Dev, a);
        std::printf("device round ok: %zu tickets, %zu chunks through a 2-buffer ring (%zu recycled before the "
                    "verdict), conflict=%d, replicas_match=%d\n",
                    tickets.size(), chunks, recycled, (int)conflict, (int)match);
        return (match && !conflict && recycled + 2 == chunks) ? 0 : 1;
    } catch (const hetm::HetmError& e) {
        std::printf("HetmError: %s\n", e.what());
        return 3;
    }
}
