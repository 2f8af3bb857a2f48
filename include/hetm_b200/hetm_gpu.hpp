// hetm_gpu.hpp — C++ binding of the hetm_b200 C-ABI for the reference HeTM tree.
//
// Header-only.  Compiled INSIDE the reference project (it includes the
// reference's own headers, proj/include/hetm/*.hpp) and linked against
// libhetm_b200.so.  It maps the ABI's int status codes back onto the
// reference's exception hierarchy (types.hpp:35-49) and accepts the
// reference's types directly:
//   * hetm::LogChunk / WriteLogEntry (bus.hpp:43-49, write_log.hpp:16-25) are
//     passed to hetm_dev_stream_chunk without copying: the 24-byte entry is
//     layout-identical to hetm_log_entry (static_assert below);
//   * BitmapSnapshot (bitmap.hpp:15-23) is filled from
//     hetm_dev_snapshot_bitmap, whose word layout is the same.
// See INTEGRATION.md for where the engine plugs it in.
#pragma once

#include <cstddef>
#include <cstdint>
#include <span>
#include <stdexcept>
#include <vector>

#include "hetm/bitmap.hpp"
#include "hetm/bus.hpp"
#include "hetm/types.hpp"
#include "hetm/write_log.hpp"
#include "hetm_b200/capi.h"

namespace hetm::b200 {

static_assert(sizeof(WriteLogEntry) == sizeof(hetm_log_entry), "wire format");
static_assert(offsetof(WriteLogEntry, addr) == offsetof(hetm_log_entry, addr));
static_assert(offsetof(WriteLogEntry, value) == offsetof(hetm_log_entry, value));
static_assert(offsetof(WriteLogEntry, ts) == offsetof(hetm_log_entry, ts));

/// Rethrows an ABI status as the reference's exception class.
inline void check(int rc) {
    const char* m = hetm_strerror(rc);
    switch (rc) {
        case HETM_OK: return;
        case HETM_ERR_INVALID_SIZE: throw InvalidSizeError(m);
        case HETM_ERR_OUT_OF_BOUNDS: throw OutOfBoundsError(m);
        case HETM_ERR_ROUND_CLOSED: throw RoundClosedError(m);
        case HETM_ERR_KERNEL_NOT_REGISTERED: throw KernelNotRegisteredError(m);
        case HETM_ERR_LIVELOCK: throw LivelockError(m);
        case HETM_ERR_NO_IMPLEMENTATION: throw NoImplementationError(m);
        case HETM_ERR_BAD_AFFINITY: throw BadAffinityError(m);
        case HETM_ERR_INCOMPLETE_TRACE: throw IncompleteTraceError(m);
        case HETM_ERR_NONDETERMINISTIC: throw NondeterministicInputError(m);
        case HETM_ERR_CONFIG: throw ConfigError(m);
        case HETM_ERR_IO: throw IoError(m);
        default: throw HetmError(m);  // CUDA / no-device / state: no CPU fallback
    }
}

/// The device guest + device half of the engine for one STMR shard.
class GpuDevice {
public:
    GpuDevice(std::size_t sizeWords, std::size_t rsGranBytes = 1024,
              std::size_t chunkBytes = ChunkMap::kDefaultChunkBytes, int device = 0,
              std::uint64_t shardBase = 0) {
        hetm_dev_config cfg;
        hetm_dev_config_default(&cfg);
        cfg.size_words = sizeWords;
        cfg.rs_gran_bytes = rsGranBytes;
        cfg.chunk_bytes = chunkBytes;
        cfg.device = device;
        cfg.shard_base = shardBase;
        check(hetm_dev_open(&cfg, &d_));
    }
    ~GpuDevice() {
        if (d_) hetm_dev_close(d_);
    }
    GpuDevice(const GpuDevice&) = delete;
    GpuDevice& operator=(const GpuDevice&) = delete;

    // stmr raw ops
    void rawWrite(Replica r, WordIdx addr, Word v) { check(hetm_dev_raw_write(d_, static_cast<int>(r), addr, v)); }
    Word rawRead(Replica r, WordIdx addr) {
        std::uint64_t v = 0;
        check(hetm_dev_raw_read(d_, static_cast<int>(r), addr, &v));
        return v;
    }

    // guest-stm-batch
    void registerKernel(int kernelId) { check(hetm_dev_register_kernel(d_, kernelId)); }
    std::vector<std::uint64_t> executeBatch(int kernelId, const void* inputs, std::size_t recBytes, std::size_t nTx,
                                            hetm_batch_stats* stats = nullptr) {
        std::vector<std::uint64_t> tickets(nTx);
        check(hetm_dev_execute_batch(d_, kernelId, inputs, recBytes, nTx, tickets.data(), stats));
        return tickets;
    }
    void clearRound(bool resetTs = false) { check(hetm_dev_clear_round(d_, resetTs ? HETM_CLEAR_RESET_TS : 0u)); }

    BitmapSnapshot snapshot(int which, std::size_t granBytes, std::size_t nBits) {
        std::uint64_t n = 0;
        check(hetm_dev_bitmap_words(d_, which, &n));
        BitmapSnapshot s{granBytes, nBits, std::vector<std::uint64_t>(n)};
        check(hetm_dev_snapshot_bitmap(d_, which, s.words.data(), n));
        return s;
    }

    // interconnect sink + engine validation (bus.hpp:78-82)
    /// Bus::streamChunk (bus.hpp:80) onto the device: returns the reference's
    /// Delivery (seq, nEntries, cost = wire bytes / the link, delivered = the H2D
    /// copy already completed) and, in *handle, the completion id to poll with
    /// delivered() / waitDelivered().  `c.entries` is borrowed until then.
    Delivery streamChunk(const LogChunk& c, bool apply = true, std::uint64_t* handle = nullptr) {
        hetm_delivery dl{};
        check(hetm_dev_stream_chunk_ex(d_, reinterpret_cast<const hetm_log_entry*>(c.entries.data()),
                                       c.entries.size(), c.sourceThread, c.seq,
                                       apply ? HETM_APPLY : HETM_VALIDATE_ONLY, &dl));
        if (handle) *handle = dl.handle;
        Delivery out;
        out.seq = dl.seq;
        out.nEntries = dl.n_entries;
        out.cost = static_cast<double>(dl.bytes);
        out.delivered = delivered(dl.handle);
        return out;
    }
    /// The chunk's entries reached the device (its host buffer may be reused).
    bool delivered(std::uint64_t handle) {
        int done = 0;
        check(hetm_dev_delivery_done(d_, handle, &done));
        return done != 0;
    }
    void waitDelivered(std::uint64_t handle) { check(hetm_dev_delivery_wait(d_, handle)); }
    /// Early-validation period k.
    void setValidationPeriod(std::uint32_t k) { check(hetm_dev_set_validation_period(d_, k)); }
    void applyLog() { check(hetm_dev_apply_log(d_)); }
    bool roundVerdict() {
        int c = 0;
        check(hetm_dev_round_verdict(d_, &c));
        return c != 0;
    }
    void closeLogIntake() { check(hetm_dev_close_intake(d_)); }

    // merge; hostReplica spans this shard's words
    /// After the host cut-off: stage the delta merge under validation and apply
    /// it speculatively (undone by the abort paths); needs HETM_CFG_MERGE_DELTA.
    void mergePrepare(std::span<Word> hostReplica) { check(hetm_dev_merge_prepare(d_, hostReplica.data())); }
    void mergeCommit(std::span<Word> hostReplica) { check(hetm_dev_merge_commit(d_, hostReplica.data(), nullptr)); }
    void mergeAbortDevice(std::span<const Word> hostReplica, bool optimized = true) {
        check(hetm_dev_merge_abort_device(d_, optimized ? 1 : 0, hostReplica.data(), nullptr));
    }
    void mergeAbortHost(std::span<Word> hostReplica, std::span<const Word> hostSnapshot) {
        check(hetm_dev_merge_abort_host(d_, hostReplica.data(), hostSnapshot.data(), nullptr));
    }
    void mergeWait() { check(hetm_dev_merge_wait(d_)); }

    /// Batch schedule: HETM_SCHED_OPTIMISTIC | HETM_SCHED_SCAN | HETM_SCHED_AUTO (default).
    void setSchedule(int mode) { check(hetm_dev_set_schedule(d_, mode)); }

    hetm_dev* handle() { return d_; }

private:
    hetm_dev* d_ = nullptr;
};

}  // namespace hetm::b200
