// host_tm.hpp — the host guest TM of SHeTM (guest-stm-word)
// and its write log (proj/include/hetm/write_log.hpp:16-101), header-only C++20.
//
// This is the CPU side of the path: host worker threads run transactions on
// the host replica with TM_begin / TM_read / TM_write / TM_commit (the HeTM
// names of the north_star; SPEC.md:123-158 begin/read/write/commit), and every
// committed update transaction hands its <addr,value,ts> write set to the
// commit callback which appends it to the calling thread's
// WriteLog.  The log is the input of the device-side validation
// (hetm_dev_stream_chunk); the entry is layout-identical to hetm_log_entry.
//
// TL2 design ("TL2-style per-word versioned locks with commit-time
// validation"): a striped table of versioned locks {version:63 | locked:1};
// begin samples the global clock (rv); a read is consistent iff its lock is
// free with version <= rv before and after the value load; commit locks the
// write set in canonical (ascending lock index) order, takes ts = ++clock,
// validates the read set against rv, publishes, and releases with version ts
// — clock advance and write-back are atomic w.r.t. other committers of the
// same words, so per-address ts order = commit order.
// Writes imply reads (no blind writes).  Aborts throw
// TxAbort (not a std::exception, types.hpp:51-54); the caller retries.
//
// Compiled against the reference headers (-I <reference>/proj/include), the
// host TM speaks the reference's own types: aborts throw ::hetm::TxAbort
// (types.hpp:54), out-of-range addresses ::hetm::OutOfBoundsError
// (types.hpp:39), and commitTo(::hetm::WriteLog&) appends committed write
// sets to the reference's WriteLog (write_log.hpp:31-101), whose entries are
// layout-identical to hetm_log_entry.  A reference worker loop written as
// `catch (hetm::TxAbort&)` therefore catches this TM's aborts.  Without those
// headers the same names are provided here.
#pragma once

#include <algorithm>
#include <atomic>
#include <cstddef>
#include <cstdint>
#include <cstring>
#include <exception>
#include <functional>
#include <memory>
#include <mutex>
#include <span>
#include <stdexcept>
#include <vector>

#include "hetm_b200/capi.h"
#include "hetm_b200/trace.hpp"

#if !defined(HETM_B200_NO_REFERENCE_TYPES) && __has_include(<hetm/types.hpp>) && __has_include(<hetm/write_log.hpp>)
#include <hetm/types.hpp>
#include <hetm/write_log.hpp>
#define HETM_B200_REFERENCE_TYPES 1
#endif

namespace hetm::b200 {

#ifdef HETM_B200_REFERENCE_TYPES
/// The reference's abort signal (types.hpp:51-54) and OutOfBoundsError (types.hpp:39).
using TxAbort = ::hetm::TxAbort;
using OutOfBoundsError = ::hetm::OutOfBoundsError;
static_assert(sizeof(::hetm::WriteLogEntry) == sizeof(hetm_log_entry) &&
                  offsetof(::hetm::WriteLogEntry, addr) == offsetof(hetm_log_entry, addr) &&
                  offsetof(::hetm::WriteLogEntry, value) == offsetof(hetm_log_entry, value) &&
                  offsetof(::hetm::WriteLogEntry, ts) == offsetof(hetm_log_entry, ts),
              "WriteLogEntry (write_log.hpp:16-21) is the 24-byte wire entry");
#else
/// Transaction abort signal (types.hpp:51-54 semantics: not a std::exception).
struct TxAbort {};
/// OutOfBoundsError (types.hpp:36-39 semantics: a runtime_error).
struct OutOfBoundsError : std::runtime_error {
    using std::runtime_error::runtime_error;
};
#endif
using HostOutOfBounds = OutOfBoundsError;  // round-1 name

/// Per-thread append-only logs, ts-ordered within a thread (write_log.hpp:27-30).
/// All threads register before a round starts (write_log.hpp:33-37 race note).
/// Same operations as the reference WriteLog (registerThread, threadCount,
/// append, entryCount, totalEntries, slice, allEntries, clearRound) over the
/// wire entry type.
class WriteLog {
public:
    explicit WriteLog(int threads = 0) : per_(threads) {
        for (auto& p : per_) p = std::make_unique<PerThread>();
    }
    /// registerThread (write_log.hpp:33-37): call before the round starts
    int registerThread() {
        per_.push_back(std::make_unique<PerThread>());
        return static_cast<int>(per_.size()) - 1;
    }
    int threadCount() const { return static_cast<int>(per_.size()); }
    int threads() const { return threadCount(); }
    std::size_t totalEntries() const {
        std::size_t n = 0;
        for (int t = 0; t < threadCount(); ++t) n += entryCount(t);
        return n;
    }
    /// slice (write_log.hpp:58-69): copies entries [from, from+max) of one thread
    std::vector<hetm_log_entry> slice(int thread, std::size_t from, std::size_t max) const {
        auto& p = *per_.at(thread);
        std::lock_guard<std::mutex> g(p.mu);
        std::vector<hetm_log_entry> out;
        if (from >= p.entries.size()) return out;
        const std::size_t end = std::min(p.entries.size(), from + max);
        out.assign(p.entries.begin() + from, p.entries.begin() + end);
        return out;
    }
    /// append (write_log.hpp:44-48)
    void append(int thread, std::span<const hetm_log_entry> es) {
        auto& p = *per_.at(thread);
        std::lock_guard<std::mutex> g(p.mu);
        p.entries.insert(p.entries.end(), es.begin(), es.end());
    }
    std::size_t entryCount(int thread) const {
        auto& p = *per_.at(thread);
        std::lock_guard<std::mutex> g(p.mu);
        return p.entries.size();
    }
    /// entries [from, min(to, size)) of one thread, copied out (write_log.hpp:63-72)
    std::size_t slice(int thread, std::size_t from, std::size_t to, hetm_log_entry* out) const {
        auto& p = *per_.at(thread);
        std::lock_guard<std::mutex> g(p.mu);
        to = std::min(to, p.entries.size());
        if (from >= to) return 0;
        std::copy(p.entries.begin() + from, p.entries.begin() + to, out);
        return to - from;
    }
    /// every entry in THREAD order (write_log.hpp:74-82)
    std::vector<hetm_log_entry> allEntries() const {
        std::vector<hetm_log_entry> out;
        for (auto& p : per_) {
            std::lock_guard<std::mutex> g(p->mu);
            out.insert(out.end(), p->entries.begin(), p->entries.end());
        }
        return out;
    }
    /// clearRound (write_log.hpp:85-91)
    void clearRound() {
        for (auto& p : per_) {
            std::lock_guard<std::mutex> g(p->mu);
            p->entries.clear();
        }
    }

private:
    struct PerThread {
        mutable std::mutex mu;
        std::vector<hetm_log_entry> entries;
    };
    std::vector<std::unique_ptr<PerThread>> per_;
};

/// The host STM over one host replica.
class HostStm {
public:
    using Callback = std::function<void(int thread, std::span<const hetm_log_entry>)>;

    struct Tx {
        uint64_t rv = 0;    // startTs
        int thread = 0;
        uint64_t id = 0;    // trace txId: thread << 40 | attempt serial number (trace on)
        std::vector<uint64_t> reads;                               // lock indices read
        std::vector<std::pair<uint64_t, uint64_t>> writes;         // addr -> pending value (insertion order)
        std::vector<std::pair<uint64_t, uint64_t>> held;           // (lock index, pre-lock word) during commit
        std::vector<hetm_log_entry> out;                           // commit scratch
    };

    HostStm(uint64_t* replica, std::size_t words, int lock_bits = 22)
        : mem_(replica), words_(words), mask_((1ull << lock_bits) - 1), locks_(new std::atomic<uint64_t>[1ull << lock_bits]) {
        for (uint64_t i = 0; i <= mask_; ++i) locks_[i].store(0, std::memory_order_relaxed);
    }

    void setCommitCallback(Callback cb) { cb_ = std::move(cb); }
    /// Checker traces: record every begin / read / write /
    /// speculative commit / abort with its value; nullptr turns recording off.
    void setTrace(Trace* t) { trace_ = t; }
    uint64_t clock() const { return clock_.load(std::memory_order_acquire); }
    /// GlobalClock floor after a device round (the device's ts space is separate; kept for completeness)
    void advanceClockTo(uint64_t v) {
        uint64_t c = clock_.load();
        while (c < v && !clock_.compare_exchange_weak(c, v)) {
        }
    }
    std::size_t sizeWords() const { return words_; }

    // ---- begin / read / write / commit
    void begin(Tx& tx, int thread) const {
        tx.rv = clock_.load(std::memory_order_acquire);
        tx.thread = thread;
        tx.reads.clear();
        tx.writes.clear();
        if (trace_) {  // ids unique over the STM's lifetime (worker threads are re-created every round)
            tx.id = (uint64_t)thread << 40 | (trace_ids_.fetch_add(1, std::memory_order_relaxed) & ((1ull << 40) - 1));
            trace_->append(0, HETM_EV_BEGIN, tx.id, 0, tx.rv);
        }
    }
    uint64_t read(Tx& tx, uint64_t addr) const {
        if (addr >= words_) throw OutOfBoundsError("host TM read out of bounds");
        for (auto it = tx.writes.rbegin(); it != tx.writes.rend(); ++it)
            if (it->first == addr) {  // read-your-writes
                if (trace_) trace_->append(0, HETM_EV_READ, tx.id, addr, it->second);
                return it->second;
            }
        const uint64_t li = lock_index(addr);
        const uint64_t l1 = locks_[li].load(std::memory_order_acquire);
        const uint64_t v = std::atomic_ref<uint64_t>(mem_[addr]).load(std::memory_order_acquire);
        const uint64_t l2 = locks_[li].load(std::memory_order_acquire);
        if ((l1 & 1) || l1 != l2 || (l1 >> 1) > tx.rv) abort_tx(tx);  // opacity: abort on stale
        tx.reads.push_back(li);
        if (trace_) trace_->append(0, HETM_EV_READ, tx.id, addr, v);
        return v;
    }
    void write(Tx& tx, uint64_t addr, uint64_t value) const {
        if (addr >= words_) throw OutOfBoundsError("host TM write out of bounds");
        struct Record {  // the WRITE event follows the implicit read in program order
            const HostStm& s;
            Tx& tx;
            uint64_t addr, value;
            ~Record() {
                if (s.trace_ && std::uncaught_exceptions() == 0) s.trace_->append(0, HETM_EV_WRITE, tx.id, addr, value);
            }
        } rec{*this, tx, addr, value};
        bool seen = false;
        for (auto& w : tx.writes)
            if (w.first == addr) {
                w.second = value;  // last write wins
                seen = true;
            }
        if (!seen) {
            (void)read(tx, addr);  // no blind writes: the implicit read
            tx.writes.emplace_back(addr, value);
        }
    }
    /// Returns the commit ts (read-only: rv, no clock advance, no callback).
    uint64_t commit(Tx& tx) {
        if (tx.writes.empty()) {  // read-only: serializes at rv
            if (trace_) trace_->append(0, HETM_EV_SPEC_COMMIT, tx.id, 0, tx.rv);
            return tx.rv;
        }
        // 1. lock the write set in canonical order
        tx.held.clear();
        for (auto& w : tx.writes) tx.held.emplace_back(lock_index(w.first), 0);
        std::sort(tx.held.begin(), tx.held.end());
        tx.held.erase(std::unique(tx.held.begin(), tx.held.end(),
                                  [](auto& a, auto& b) { return a.first == b.first; }),
                      tx.held.end());
        std::size_t got = 0;
        for (; got < tx.held.size(); ++got) {
            auto& lk = locks_[tx.held[got].first];
            uint64_t cur = lk.load(std::memory_order_relaxed);
            int spins = 0;
            while ((cur & 1) || !lk.compare_exchange_weak(cur, cur | 1, std::memory_order_acquire)) {
                if (++spins > 64) break;  // bounded spin, then abort (caller retries)
                cur = lk.load(std::memory_order_relaxed);
            }
            if (spins > 64) break;
            tx.held[got].second = cur;
        }
        if (got < tx.held.size()) {
            release(tx, got, false, 0);
            abort_tx(tx);
        }
        // 2. ts = ++clock (unique; the write locks are held)
        const uint64_t ts = clock_.fetch_add(1, std::memory_order_acq_rel) + 1;
        // 3. validate the read set against rv
        if (ts != tx.rv + 1) {
            for (uint64_t li : tx.reads) {
                const uint64_t l = locks_[li].load(std::memory_order_acquire);
                uint64_t ver = l >> 1;
                if (l & 1) {
                    auto h = std::lower_bound(tx.held.begin(), tx.held.end(), std::make_pair(li, uint64_t(0)));
                    if (h == tx.held.end() || h->first != li) {
                        release(tx, tx.held.size(), false, 0);
                        abort_tx(tx);
                    }
                    ver = h->second >> 1;
                }
                if (ver > tx.rv) {
                    release(tx, tx.held.size(), false, 0);
                    abort_tx(tx);
                }
            }
        }
        // 4. publish, release with version ts, callback with <addr,value,ts>
        tx.out.clear();
        for (auto& w : tx.writes) {
            std::atomic_ref<uint64_t>(mem_[w.first]).store(w.second, std::memory_order_release);
            tx.out.push_back(hetm_log_entry{w.first, w.second, ts});
        }
        release(tx, tx.held.size(), true, ts);
        if (trace_) trace_->append(0, HETM_EV_SPEC_COMMIT, tx.id, 0, ts);
        if (cb_) cb_(tx.thread, tx.out);
        return ts;
    }

    /// Runs `body(tx)` until it commits; returns the commit ts.
    template <class Body>
    uint64_t atomically(int thread, Body&& body) {
        Tx& tx = scratch();
        for (;;) {
            begin(tx, thread);
            try {
                body(tx);
                return commit(tx);
            } catch (const TxAbort&) {
                aborts_.fetch_add(1, std::memory_order_relaxed);
            }
        }
    }
    uint64_t aborts() const { return aborts_.load(); }

private:
    [[noreturn]] void abort_tx(Tx& tx) const {
        if (trace_) trace_->append(0, HETM_EV_ABORT, tx.id, 0, HETM_ABORT_CONFLICT);
        throw TxAbort{};
    }
    uint64_t lock_index(uint64_t addr) const { return (addr * 0x9e3779b97f4a7c15ull >> 20) & mask_; }
    void release(Tx& tx, std::size_t n, bool committed, uint64_t ts) const {
        for (std::size_t k = 0; k < n; ++k)
            locks_[tx.held[k].first].store(committed ? (ts << 1) : tx.held[k].second, std::memory_order_release);
    }
    static Tx& scratch() {
        thread_local Tx tx;
        return tx;
    }

    uint64_t* mem_;
    std::size_t words_;
    uint64_t mask_;
    std::unique_ptr<std::atomic<uint64_t>[]> locks_;
    std::atomic<uint64_t> clock_{0};
    std::atomic<uint64_t> aborts_{0};
    Callback cb_;
    Trace* trace_ = nullptr;
    mutable std::atomic<uint64_t> trace_ids_{0};
};

/// Commit callback appending each committed write set to a WriteLog
/// (write_log.hpp:44 append(thread, span)).
inline HostStm::Callback commitTo(WriteLog& log) {
    return [&log](int thread, std::span<const hetm_log_entry> es) { log.append(thread, es); };
}
#ifdef HETM_B200_REFERENCE_TYPES
/// The same into the reference's own hetm::WriteLog (entries are layout-identical).
inline HostStm::Callback commitTo(::hetm::WriteLog& log) {
    return [&log](int thread, std::span<const hetm_log_entry> es) {
        log.append(thread, std::span<const ::hetm::WriteLogEntry>(
                               reinterpret_cast<const ::hetm::WriteLogEntry*>(es.data()), es.size()));
    };
}
#endif

// Log access used by the round controller, for this WriteLog and (with the
// reference headers) the reference's hetm::WriteLog.
inline int log_threads(const WriteLog& l) { return l.threadCount(); }
inline std::size_t log_count(const WriteLog& l, int t) { return l.entryCount(t); }
inline std::size_t log_copy(const WriteLog& l, int t, std::size_t from, std::size_t n, hetm_log_entry* out) {
    return l.slice(t, from, from + n, out);
}
inline std::vector<hetm_log_entry> log_all(const WriteLog& l) { return l.allEntries(); }
inline void log_clear(WriteLog& l) { l.clearRound(); }
#ifdef HETM_B200_REFERENCE_TYPES
inline int log_threads(const ::hetm::WriteLog& l) { return l.threadCount(); }
inline std::size_t log_count(const ::hetm::WriteLog& l, int t) { return l.entryCount(t); }
inline std::size_t log_copy(const ::hetm::WriteLog& l, int t, std::size_t from, std::size_t n, hetm_log_entry* out) {
    const auto v = l.slice(t, from, n);
    std::memcpy(out, v.data(), v.size() * sizeof(hetm_log_entry));
    return v.size();
}
inline std::vector<hetm_log_entry> log_all(const ::hetm::WriteLog& l) {
    const auto v = l.allEntries();
    std::vector<hetm_log_entry> out(v.size());
    std::memcpy(out.data(), v.data(), v.size() * sizeof(hetm_log_entry));
    return out;
}
inline void log_clear(::hetm::WriteLog& l) { l.clearRound(); }
#endif

// ---- the HeTM host API names (north_star: TM_begin / TM_read / TM_write / TM_commit)
inline void TM_begin(HostStm& stm, HostStm::Tx& tx, int thread) { stm.begin(tx, thread); }
inline uint64_t TM_read(HostStm& stm, HostStm::Tx& tx, uint64_t addr) { return stm.read(tx, addr); }
inline void TM_write(HostStm& stm, HostStm::Tx& tx, uint64_t addr, uint64_t v) { stm.write(tx, addr, v); }
inline uint64_t TM_commit(HostStm& stm, HostStm::Tx& tx) { return stm.commit(tx); }

}  // namespace hetm::b200
