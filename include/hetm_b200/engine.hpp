// engine.hpp — the SHeTM round controller on the host (SPEC.md:314-433,
// engine.runRound), header-only C++20 over the C-ABI.
//
// One synchronization round (call stack SURVEY.md §3 (1)):
//   EXECUTION   the GPU-controller thread runs one device batch
//               (hetm_dev_execute_batch) while host worker threads run
//               transactions on the host replica through HostStm; their
//               commit callbacks append to the per-thread WriteLog.  The
//               streamer (the calling thread) ships every full chunk of a
//               thread's log over PCIe as it fills (hetm_dev_stream_chunk,
//               VALIDATE_ONLY = early validation) and stops
//               the host early when the device reports a conflict.
//   VALIDATION  host cut-off, the log tail streamed in APPLY mode, the early
//               chunks re-validated and applied (hetm_dev_apply_log), verdict.
//   MERGE       no conflict: mergeCommit (device write set -> host replica);
//               conflict: FavorHost mergeAbortDevice, or
//               FavorDevice mergeAbortHost: every chunk is
//               validate-only until the verdict, the host replica is restored
//               from the round-start snapshot and takes the device's chunks.
// Starvation guard: under FavorHost, after starvation_k
// consecutive DeviceAborted rounds the next round admits only read-only host
// transactions (RoundContext::updates_allowed), so the device commits.
// Chunk buffers come from a pinned staging ring (hetm_host_alloc) and are
// reused once their chunk is delivered (hetm_dev_stream_chunk_ex handle).
#pragma once

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <functional>
#include <stdexcept>
#include <string>
#include <thread>
#include <tuple>
#include <vector>

#include "hetm_b200/capi.h"
#include "hetm_b200/host_tm.hpp"
#include "hetm_b200/trace.hpp"

namespace hetm::b200 {

enum class Policy { FavorHost, FavorDevice };  // PolicyConfig.mode
enum class Outcome { Commit, DeviceAborted, HostAborted };

struct EngineConfig {
    Policy policy = Policy::FavorHost;
    uint32_t starvation_k = 3;          // PolicyConfig.starvationK (>= 1)
    uint64_t chunk_entries = 1u << 16;  // entries per streamed LogChunk
    bool early_validation = true;       // stream chunks VALIDATE_ONLY during execution
    uint32_t ev_period = 8;             // early validation every k streamed chunks
    // hostCutoff: after the execution phase the host keeps
    // committing while more than cutoff_chunks chunks of its log remain
    // undelivered to the device; 0 = the basic algorithm (the host stops when
    // the execution phase ends).  Default 4.
    uint32_t cutoff_chunks = 4;
    // Bus real-delay mode (bus.hpp:33-39 BusConfig): each streamed chunk also
    // sleeps (latency + bytes / bytes_per_unit) * real_delay_us_per_unit us, a
    // slow-link model for end-to-end experiments (0 = off: the real PCIe only).
    double bus_latency_units = 2.0;
    double bus_bytes_per_unit = 8192.0;
    double bus_real_delay_us_per_unit = 0.0;
    bool optimized_abort = true;        // mergeAbortDevice: shadow + log (true) or chunk copy (false)
    bool keep_round_log = false;        // keep a copy of the last round's host log (checkers)
    bool early_merge = true;            // stage + speculatively apply the delta merge after execution
                                        // (hetm_dev_merge_prepare; a no-op without HETM_CFG_MERGE_DELTA)
    bool pipeline_merge = false;        // a committed round returns before its merge has landed in the
                                        // host replica: the next round's device batches start under it
                                        // and its host workers wait for it (drain() before
                                        // reading the host replica outside a round)
    uint32_t fault = 0;                 // ENGINE_FAULT_* (checker mutation suite only)
};

// Engine-level mutations for the checker's mutation suite; the
// device-level ones are hetm_dev_set_fault.  Never set outside tests.
constexpr uint32_t ENGINE_FAULT_EARLY_DEVICE_COMMIT = 1;  // report device commits final before validation
constexpr uint32_t ENGINE_FAULT_DROP_CHUNK = 2;           // drop the round's first streamed log chunk

struct RoundReport {
    uint64_t round_id = 0;
    Outcome outcome = Outcome::Commit;
    bool updates_allowed = true;    // false: starvation-guard round (read-only host)
    bool conflict = false;
    bool cut_short = false;         // early validation ended the execution phase
    uint64_t host_commits = 0;
    uint64_t dev_committed = 0;
    uint64_t log_entries = 0;
    uint64_t chunks = 0;
    uint64_t bytes_merge = 0;       // merge / rollback transfer bytes (D2H + H2D + D2D)
    uint32_t dev_batches = 0;       // device batches executed in the execution phase
    uint64_t cutoff_chunks = 0;     // chunks streamed while the host ran past the execution phase
    double exec_ms = 0, validate_ms = 0, merge_ms = 0;
    double host_blocked_ms = 0;     // host admission paused (hostCutoff) until the round ended
    hetm_batch_stats batch{};

    /// (name, value, is_string) in the fixed SPEC.md:427 field order; json()
    /// and csvRow() print the same strings.
    std::vector<std::tuple<const char*, std::string, bool>> fields() const {
        static const char* names[] = {"Commit", "DeviceAborted", "HostAborted"};
        const auto u = [](uint64_t v) { return std::to_string(v); };
        const auto ms = [](double v) {
            char b[32];
            std::snprintf(b, sizeof b, "%.3f", v);
            return std::string(b);
        };
        return {{"roundId", u(round_id), false},
                {"outcome", names[(int)outcome], true},
                {"txCommittedHost", u(outcome == Outcome::HostAborted ? 0 : host_commits), false},
                {"txCommittedDev", u(outcome == Outcome::DeviceAborted ? 0 : dev_committed), false},
                {"txWastedDev", u(outcome == Outcome::DeviceAborted ? dev_committed : 0), false},
                {"bytesLogs", u(log_entries * sizeof(hetm_log_entry)), false},
                {"bytesMerge", u(bytes_merge), false},
                {"readOnlyHost", u(!updates_allowed), false},
                {"cutShort", u(cut_short), false},
                {"devBatches", u(dev_batches), false},
                {"execMs", ms(exec_ms), false},
                {"validateMs", ms(validate_ms), false},
                {"mergeMs", ms(merge_ms), false}};
    }
    std::string json() const { return json_object(fields()); }
    std::string csvRow() const { return csv_line(fields(), false); }
    static std::string csvHeader() { return csv_line(RoundReport{}.fields(), true); }

    template <class F>
    static std::string json_object(const F& fs) {
        std::string o = "{";
        for (const auto& [k, v, str] : fs) {
            if (o.size() > 1) o += ", ";
            o += std::string("\"") + k + "\": " + (str ? "\"" + v + "\"" : v);
        }
        return o + "}";
    }
    template <class F>
    static std::string csv_line(const F& fs, bool header) {
        std::string o;
        for (const auto& [k, v, str] : fs) o += (o.empty() ? "" : ",") + (header ? std::string(k) : v);
        return o;
    }
};

/// Run summary over the rounds (throughput = sum committed / sum time).
struct RunSummary {
    uint64_t rounds = 0, tx_host = 0, tx_dev = 0, tx_wasted_dev = 0, bytes_logs = 0, bytes_merge = 0;
    double time_ms = 0;
    explicit RunSummary(const std::vector<RoundReport>& rs) {
        for (const auto& r : rs) {
            ++rounds;
            tx_host += r.outcome == Outcome::HostAborted ? 0 : r.host_commits;
            tx_dev += r.outcome == Outcome::DeviceAborted ? 0 : r.dev_committed;
            tx_wasted_dev += r.outcome == Outcome::DeviceAborted ? r.dev_committed : 0;
            bytes_logs += r.log_entries * sizeof(hetm_log_entry);
            bytes_merge += r.bytes_merge;
            // each phase rounded like the per-round rows, so the summary recomputes from them exactly
            for (double m : {r.exec_ms, r.validate_ms, r.merge_ms}) time_ms += std::round(m * 1000.0) / 1000.0;
        }
    }
    std::vector<std::tuple<const char*, std::string, bool>> fields() const {
        const auto u = [](uint64_t v) { return std::to_string(v); };
        char t[32], thr[48];
        std::snprintf(t, sizeof t, "%.3f", time_ms);
        std::snprintf(thr, sizeof thr, "%.1f", time_ms > 0 ? (tx_host + tx_dev) / (time_ms * 1e-3) : 0.0);
        return {{"rounds", u(rounds), false},           {"txCommittedHost", u(tx_host), false},
                {"txCommittedDev", u(tx_dev), false},     {"txWastedDev", u(tx_wasted_dev), false},
                {"bytesLogs", u(bytes_logs), false},      {"bytesMerge", u(bytes_merge), false},
                {"timeMs", t, false},                     {"throughputTxPerS", thr, false}};
    }
};

/// emitReport: one row per round in a deterministic field
/// order plus a summary block; "csv" or "json"; throws on an I/O error.
inline void emitReport(const std::vector<RoundReport>& rounds, const std::string& format, const std::string& path) {
    std::string out;
    const RunSummary sum(rounds);
    if (format == "csv") {
        out = RoundReport::csvHeader() + "\n";
        for (const auto& r : rounds) out += r.csvRow() + "\n";
        out += "\n" + RoundReport::csv_line(sum.fields(), true) + "\n" + RoundReport::csv_line(sum.fields(), false) + "\n";
    } else if (format == "json") {
        out = "{\"rounds\": [";
        for (std::size_t i = 0; i < rounds.size(); ++i) out += (i ? ", " : "") + rounds[i].json();
        out += "], \"summary\": " + RoundReport::json_object(sum.fields()) + "}\n";
    } else {
        throw std::invalid_argument("emitReport: format is csv or json");
    }
    FILE* f = std::fopen(path.c_str(), "wb");
    if (!f) throw std::runtime_error("emitReport: io-error opening " + path);
    const bool ok = std::fwrite(out.data(), 1, out.size(), f) == out.size();
    if (std::fclose(f) != 0 || !ok) throw std::runtime_error("emitReport: io-error writing " + path);
}

/// What a host worker sees of the round.
struct RoundContext {
    const std::atomic<bool>& stop;  // host cut-off / early-validation stop
    bool updates_allowed;           // false under the starvation guard: read-only transactions only
};

inline void check_rc(int rc, const char* what) {
    if (rc != HETM_OK) throw std::runtime_error(std::string(what) + ": " + hetm_strerror(rc));
}

/// The round controller over a write log: this library's WriteLog or, with the
/// reference headers, the reference's hetm::WriteLog (log_* in host_tm.hpp).
template <class Log>
class BasicEngine {
public:
    BasicEngine(hetm_dev* dev, HostStm& stm, Log& log, uint64_t* host_replica, EngineConfig cfg = {})
        : dev_(dev), stm_(stm), log_(log), host_(host_replica), cfg_(cfg), shipped_(log_threads(log), 0) {
        if (cfg_.starvation_k < 1) throw std::invalid_argument("starvationK >= 1 (SPEC.md:332)");
        if (cfg_.ev_period < 1) throw std::invalid_argument("early-validation period k >= 1 (SPEC.md:423)");
        if (cfg_.policy == Policy::FavorDevice) snapshot_.resize(stm.sizeWords());
        check_rc(hetm_dev_set_validation_period(dev_, cfg_.ev_period), "set_validation_period");
    }
    ~BasicEngine() {
        for (auto& b : pool_) hetm_host_free(b.ptr);
    }
    /// pipeline_merge: wait until the last committed round's merge has landed in
    /// the host replica (before reading it outside a round).
    void drain() {
        if (merge_pending_) {
            check_rc(hetm_dev_merge_wait(dev_), "merge_wait");
            merge_pending_ = false;
        }
    }

    /// Pinned staging buffers allocated so far (chunks recycle them once delivered).
    std::size_t stagingBuffers() const { return pool_.size(); }

    /// Host worker: run transactions until ctx.stop is set or its work ends
    /// (read-only ones when !ctx.updates_allowed); returns how many committed.
    using HostWorker = std::function<uint64_t(int thread, const RoundContext& ctx)>;
    uint32_t consecutiveDeviceAborts() const { return dev_aborts_; }

    /// Checker traces: host transactions through HostStm,
    /// device batches through hetm_dev_trace_next_batch (bank and rw kernels),
    /// round markers and the final-commit / abort verdict of every speculative
    /// commit.  nullptr turns recording off.
    void setTrace(Trace* t) {
        trace_ = t;
        stm_.setTrace(t);
    }

    /// Next device batch of the round: fill inputs/n_tx/tickets_out and return
    /// true, or return false when the execution budget is spent.
    struct Batch {
        const void* inputs = nullptr;
        uint64_t n_tx = 0;
        uint64_t* tickets_out = nullptr;
    };
    using BatchSource = std::function<bool(uint32_t k, Batch& b)>;

    /// One round with a single device batch.
    RoundReport runRound(int kernel_id, const void* inputs, uint64_t rec_bytes, uint64_t n_tx, uint64_t* tickets_out,
                         const HostWorker& worker) {
        return runRoundBatches(kernel_id, rec_bytes, [&](uint32_t k, Batch& b) {
            if (k) return false;
            b = Batch{inputs, n_tx, tickets_out};
            return true;
        }, worker);
    }

    /// One round whose execution phase runs device batches back to back until
    /// `next` ends the budget — or until early validation finds a conflict, which
    /// ends the phase before the next batch is launched.
    RoundReport runRoundBatches(int kernel_id, uint64_t rec_bytes, const BatchSource& next,
                                const HostWorker& worker) {
        RoundReport rep;
        rep.round_id = round_id_++;
        if (trace_) trace_->beginRound((uint32_t)rep.round_id);
        dropped_ = false;
        const bool favor_device = cfg_.policy == Policy::FavorDevice;
        // starvation guard (FavorHost): a read-only host round after K device aborts
        rep.updates_allowed = favor_device || dev_aborts_ < cfg_.starvation_k;
        // a pipelined merge of the previous round lands before anything on the host reads the replica
        // (the FavorDevice snapshot, the host workers); the device batches below do not wait for it
        const bool merge_pending = merge_pending_;
        merge_pending_ = false;
        if (favor_device && merge_pending) check_rc(hetm_dev_merge_wait(dev_), "merge_wait");
        // FavorDevice: explicit host snapshot at round start
        if (favor_device) std::memcpy(snapshot_.data(), host_, snapshot_.size() * sizeof(uint64_t));
        const int stream_mode = (favor_device || cfg_.early_validation) ? HETM_VALIDATE_ONLY : HETM_APPLY;
        const auto t0 = std::chrono::steady_clock::now();
        std::atomic<bool> stop{false}, gpu_done{false};
        const RoundContext ctx{stop, rep.updates_allowed};
        int gpu_rc = HETM_OK;
        // ---- EXECUTION
        std::atomic<bool> cut{false};
        std::thread gpu([&] {  // GPU-controller: batches until the budget ends or a conflict shows
            Batch b;
            for (uint32_t k = 0; !cut.load(std::memory_order_acquire) && next(k, b); ++k) {
                hetm_batch_stats st{};
                if (trace_) {
                    trace_rec_.assign(b.n_tx * HETM_TRACE_TX_WORDS, ~0ull);
                    gpu_rc = hetm_dev_trace_next_batch(dev_, trace_rec_.data());
                    if (gpu_rc != HETM_OK) break;
                }
                gpu_rc = hetm_dev_execute_batch(dev_, kernel_id, b.inputs, rec_bytes, b.n_tx, b.tickets_out, &st);
                if (gpu_rc != HETM_OK) break;
                if (trace_) trace_batch(kernel_id, b);
                rep.batch = st;
                rep.dev_committed += st.committed;
                ++rep.dev_batches;
            }
            gpu_done.store(true, std::memory_order_release);
        });
        std::vector<std::thread> hosts;
        std::vector<uint64_t> commits(log_threads(log_), 0);
        if (merge_pending && !favor_device) check_rc(hetm_dev_merge_wait(dev_), "merge_wait");  // GPU already running
        for (int t = 0; t < log_threads(log_); ++t)
            hosts.emplace_back([&, t] { commits[t] = worker(t, ctx); });
        while (!gpu_done.load(std::memory_order_acquire)) {
            stream_full_chunks(stream_mode, rep, &gpu_done);  // the execution phase's end is noticed between chunks
            int c = 0;
            if (cfg_.early_validation && !rep.cut_short && hetm_dev_poll_conflict(dev_, &c) == HETM_OK && c) {
                // a conflict already decides the round: FavorHost dooms the device's
                // batches (launch no more), FavorDevice dooms the host's transactions (stop them)
                rep.cut_short = true;
                if (favor_device) stop.store(true, std::memory_order_release);
                else cut.store(true, std::memory_order_release);
            }
            std::this_thread::sleep_for(std::chrono::microseconds(50));
        }
        gpu.join();
        const auto t1 = std::chrono::steady_clock::now();
        // ---- VALIDATION: the log tail (APPLY, or validate-only under FavorDevice),
        // early chunks re-validated + applied (FavorDevice: only on success)
        const int tail_mode = favor_device ? HETM_VALIDATE_ONLY : HETM_APPLY;
        // hostCutoff: the host keeps committing while the log
        // streams, and pauses once at most cutoff_chunks chunks are undelivered;
        // 0 stops it as the execution phase ends (the basic algorithm).  Not
        // after an early conflict: the round is decided, FavorDevice stopped
        // the host already.
        // The window also ends once it has shipped as many chunks as were
        // undelivered when execution ended (what the basic algorithm ships with
        // the host blocked), so a producer faster than the link cannot extend
        // the round without bound.
        if (cfg_.cutoff_chunks > 0 && gpu_rc == HETM_OK && !rep.cut_short && rep.updates_allowed) {
            const uint64_t backlog0 = backlog_chunks();
            while (backlog_chunks() > cfg_.cutoff_chunks && rep.cutoff_chunks < backlog0) {
                const uint64_t before = rep.chunks;
                stream_all(tail_mode, rep);  // partial chunks too: the backlog drains
                rep.cutoff_chunks += rep.chunks - before;
                if (rep.chunks == before) std::this_thread::sleep_for(std::chrono::microseconds(20));
            }
        }
        stop.store(true, std::memory_order_release);  // host admission paused until the merge completes
        const auto t_block = std::chrono::steady_clock::now();
        for (auto& h : hosts) h.join();
        check_rc(gpu_rc, "executeBatch");
        for (uint64_t c : commits) rep.host_commits += c;
        // the host is paused and the device batches are done: the device write
        // set can travel to the host replica now, under the validation phase
        // (undone by the abort paths if the round does not commit)
        if (cfg_.early_merge) check_rc(hetm_dev_merge_prepare(dev_, host_), "merge_prepare");
        stream_full_chunks(tail_mode, rep);
        stream_tail(rep, tail_mode);
        int conflict = 0;
        if (!favor_device) check_rc(hetm_dev_apply_log(dev_), "apply_log");
        check_rc(hetm_dev_round_verdict(dev_, &conflict), "round_verdict");
        rep.conflict = conflict != 0;
        if (favor_device && !rep.conflict) {
            check_rc(hetm_dev_apply_log(dev_), "apply_log");
            check_rc(hetm_dev_round_verdict(dev_, &conflict), "round_verdict");
        }
        const auto t2 = std::chrono::steady_clock::now();
        // ---- MERGE (the trace records the verdict of every speculative commit)
        if (trace_) {
            const bool early = (cfg_.fault & ENGINE_FAULT_EARLY_DEVICE_COMMIT) != 0;
            trace_->finalizeRound(!rep.conflict || !favor_device, !rep.conflict || favor_device || early);
        }
        if (!rep.conflict) {
            rep.outcome = Outcome::Commit;
            hetm_merge_stats ms{};
            check_rc(hetm_dev_merge_commit(dev_, host_, &ms), "merge_commit");
            rep.bytes_merge = ms.bytes_d2h + ms.bytes_h2d + ms.bytes_d2d;
            if (cfg_.pipeline_merge) merge_pending_ = true;  // lands under the next round's device batches
            else check_rc(hetm_dev_merge_wait(dev_), "merge_wait");
            dev_aborts_ = 0;
        } else if (!favor_device) {
            rep.outcome = Outcome::DeviceAborted;
            hetm_merge_stats ms{};
            check_rc(hetm_dev_merge_abort_device(dev_, cfg_.optimized_abort ? 1 : 0, host_, &ms),
                     "merge_abort_device");
            rep.bytes_merge = ms.bytes_d2h + ms.bytes_h2d + ms.bytes_d2d;
            ++dev_aborts_;
        } else {
            rep.outcome = Outcome::HostAborted;
            hetm_merge_stats ms{};
            check_rc(hetm_dev_merge_abort_host(dev_, host_, snapshot_.data(), &ms), "merge_abort_host");
            rep.bytes_merge = ms.bytes_d2h + ms.bytes_h2d + ms.bytes_d2d;
            check_rc(hetm_dev_merge_wait(dev_), "merge_wait");
        }
        check_rc(hetm_dev_clear_round(dev_, 0), "clear_round");
        if (cfg_.keep_round_log) last_log_ = log_all(log_);
        log_clear(log_);
        std::fill(shipped_.begin(), shipped_.end(), 0);
        const auto t3 = std::chrono::steady_clock::now();
        rep.host_blocked_ms = std::chrono::duration<double, std::milli>(t3 - t_block).count();
        rep.exec_ms = std::chrono::duration<double, std::milli>(t1 - t0).count();
        rep.validate_ms = std::chrono::duration<double, std::milli>(t2 - t1).count();
        rep.merge_ms = std::chrono::duration<double, std::milli>(t3 - t2).count();
        return rep;
    }

    /// The last round's host log in WriteLog::allEntries order (keep_round_log).
    const std::vector<hetm_log_entry>& lastRoundLog() const { return last_log_; }

private:
    // Pinned staging ring: a buffer is reused as soon as the chunk it carried is
    // delivered (hetm_dev_delivery_done), so the pool stays at the chunks in
    // flight instead of the whole round's log.
    struct Staging {
        void* ptr = nullptr;
        uint64_t handle = 0;
        bool busy = false;
    };
    std::size_t chunk_buffer() {
        for (std::size_t k = 0; k < pool_.size(); ++k) {
            const std::size_t idx = (ring_ + k) % pool_.size();
            Staging& b = pool_[idx];
            int done = 1;
            if (b.busy) check_rc(hetm_dev_delivery_done(dev_, b.handle, &done), "delivery_done");
            if (done) {
                b.busy = false;
                ring_ = (idx + 1) % pool_.size();
                return idx;
            }
        }
        Staging b;
        check_rc(hetm_host_alloc(cfg_.chunk_entries * sizeof(hetm_log_entry), &b.ptr), "host_alloc");
        pool_.push_back(b);
        return pool_.size() - 1;
    }
    // chunks of the host log not yet delivered to the device: shipped but in
    // flight, plus the unshipped entries of every thread (a partial one counts)
    uint64_t backlog_chunks() {
        uint64_t n = 0;
        for (auto& b : pool_) {
            int done = 1;
            if (b.busy) check_rc(hetm_dev_delivery_done(dev_, b.handle, &done), "delivery_done");
            if (done) b.busy = false;
            else ++n;
        }
        for (int t = 0; t < log_threads(log_); ++t)
            n += (log_count(log_, t) - shipped_[t] + cfg_.chunk_entries - 1) / cfg_.chunk_entries;
        return n;
    }
    // Device events of one traced batch, in program order per transaction.
    void trace_batch(int kernel_id, const Batch& b) {
        const uint64_t batch = trace_batches_++;
        for (uint64_t i = 0; i < b.n_tx; ++i) {
            const uint64_t* r = trace_rec_.data() + i * HETM_TRACE_TX_WORDS;
            if (r[0] == ~0ull) continue;  // did not commit
            const uint64_t id = 1ull << 63 | batch << 32 | i;
            trace_->append(1, HETM_EV_BEGIN, id, 0, 0);
            if (kernel_id == HETM_KERNEL_BANK) {
                const hetm_bank_tx& t = static_cast<const hetm_bank_tx*>(b.inputs)[i];
                for (int k = 0; k < 4; ++k) trace_->append(1, HETM_EV_READ, id, t.acct[k], r[1 + k]);
                for (int k = 0; k < 2; ++k) trace_->append(1, HETM_EV_WRITE, id, t.acct[k], r[7 + k]);
            } else if (kernel_id == HETM_KERNEL_RW) {
                const hetm_rw_tx& t = static_cast<const hetm_rw_tx*>(b.inputs)[i];
                for (uint32_t k = 0; k < std::min<uint32_t>(t.nr, 4); ++k)
                    trace_->append(1, HETM_EV_READ, id, t.r_addr[k], r[1 + k]);
                for (uint32_t k = 0; k < std::min<uint32_t>(t.nw, 2); ++k) {
                    trace_->append(1, HETM_EV_READ, id, t.w_addr[k], r[5 + k]);
                    trace_->append(1, HETM_EV_WRITE, id, t.w_addr[k], r[7 + k]);
                }
            }
            trace_->append(1, HETM_EV_SPEC_COMMIT, id, 0, r[0]);
        }
    }
    void ship(int t, uint64_t n, int mode, RoundReport& rep) {
        Staging& b = pool_[chunk_buffer()];
        hetm_log_entry* buf = static_cast<hetm_log_entry*>(b.ptr);
        const uint64_t got = log_copy(log_, t, shipped_[t], n, buf);
        if ((cfg_.fault & ENGINE_FAULT_DROP_CHUNK) && !dropped_ && got) {  // mutation: the chunk never reaches the GPU
            dropped_ = true;
            shipped_[t] += got;
            return;
        }
        hetm_delivery dl{};
        check_rc(hetm_dev_stream_chunk_ex(dev_, buf, got, t, seq_++, mode, &dl), "stream_chunk");
        b.handle = dl.handle;
        b.busy = true;
        shipped_[t] += got;
        rep.log_entries += got;
        ++rep.chunks;
        if (cfg_.bus_real_delay_us_per_unit > 0) {  // BusConfig real-delay mode (bus.hpp:37-39)
            const double cost = cfg_.bus_latency_units + double(got * sizeof(hetm_log_entry)) / cfg_.bus_bytes_per_unit;
            std::this_thread::sleep_for(std::chrono::duration<double, std::micro>(cost * cfg_.bus_real_delay_us_per_unit));
        }
    }
    void stream_full_chunks(int mode, RoundReport& rep, const std::atomic<bool>* until = nullptr) {
        for (int t = 0; t < log_threads(log_); ++t)
            while (log_count(log_, t) - shipped_[t] >= cfg_.chunk_entries) {
                if (until && until->load(std::memory_order_acquire)) return;
                ship(t, cfg_.chunk_entries, mode, rep);
            }
    }
    // every unshipped entry, in chunks of at most chunk_entries (host workers
    // may still be appending during the hostCutoff window)
    void stream_tail(RoundReport& rep, int mode) {
        for (int t = 0; t < log_threads(log_); ++t) {
            const uint64_t end = log_count(log_, t);
            while (end > shipped_[t]) ship(t, std::min<uint64_t>(end - shipped_[t], cfg_.chunk_entries), mode, rep);
        }
    }
    void stream_all(int mode, RoundReport& rep) {
        stream_full_chunks(mode, rep);
        stream_tail(rep, mode);
    }

    hetm_dev* dev_;
    HostStm& stm_;
    Log& log_;
    uint64_t* host_;
    EngineConfig cfg_;
    std::vector<uint64_t> shipped_;
    std::vector<Staging> pool_;
    std::size_t ring_ = 0;
    uint64_t seq_ = 0;
    std::vector<hetm_log_entry> last_log_;
    std::vector<uint64_t> snapshot_;  // FavorDevice round-start host snapshot
    uint64_t round_id_ = 0;
    uint32_t dev_aborts_ = 0;         // consecutiveDeviceAborts
    bool merge_pending_ = false;      // pipeline_merge: the last committed round's merge has not landed yet
    Trace* trace_ = nullptr;
    std::vector<uint64_t> trace_rec_;  // per-batch device trace records
    uint64_t trace_batches_ = 0;
    bool dropped_ = false;             // ENGINE_FAULT_DROP_CHUNK: this round's chunk is gone
};

using Engine = BasicEngine<WriteLog>;

}  // namespace hetm::b200
