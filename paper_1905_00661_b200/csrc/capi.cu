// capi.cu — the hetm_b200 C-ABI (include/hetm_b200/capi.h): device handle,
// round state, streams, log arena, merge paths.
//
// Stream layout (one handle = one GPU = one STMR shard):
//   s_exec   batch transaction kernels (execution phase)
//   s_copy   H2D log chunk copies (interconnect streamChunk)
//   s_val    validation kernels; APPLY kernels wait on the tail of s_exec
//   s_merge  shadow update, delta sort/gather, rollback, round clear
//   s_d2h    merge device->host copies (chunks from devShadow, or the delta
//            records), overlapping the next round's execution (double
//            buffering)
//   s_zc     zero-copy delta stores into the mapped host replica (optional)
//   s_in     input pieces H2D of a host-buffer batch, under the kernel on the
//            previous piece; s_out its tickets / results D2H
//   s_est    the AUTO schedule's hot-spot estimate of device-pointer batches
//   s_win    (HETM_WIN_SIDE=1) merge_stage's devShadow patch with the host-log
//            winners, beside the pick/emit on s_merge (joined before ev_shadow)
// plus the worker pool that scatters the merge delta into the host replica as
// its pieces land.  Events carry every cross-stream dependency; nothing blocks
// the host except the explicitly synchronous calls (verdict, merge_wait,
// snapshots, stats) and the pool hand-off of merge_prepare.
#include <algorithm>
#include <array>
#include <atomic>
#include <chrono>
#include <condition_variable>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <map>
#include <memory>
#include <mutex>
#include <thread>
#include <set>
#include <string>
#include <utility>
#include <vector>

#include <sched.h>
#include <sys/mman.h>

#include <nvtx3/nvToolsExt.h>

#include "common.cuh"
#include "device_tm.cuh"
#include "kernels.h"

namespace hetm_b200 {
int query_tx_occupancy(int* blocks);
int query_val_occupancy(int* blocks);
}  // namespace hetm_b200

using namespace hetm_b200;

namespace {
// NVTX range per round phase (execute / stream / verdict / merge / clear /
// exchange) for nsys timelines; header-only nvtx3, no-ops without a tool.
struct NvtxRange {
    explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
    ~NvtxRange() { nvtxRangePop(); }
};

// Persistent host workers for the delta merge: start(f) runs f(w, n) once on
// every worker w in [0, n) and returns immediately; wait() joins that job.
class WorkerPool {
public:
    explicit WorkerPool(int n) : n_(n) {
        for (int w = 0; w < n; ++w) th_.emplace_back([this, w] { loop(w); });
    }
    ~WorkerPool() {
        {
            std::lock_guard<std::mutex> g(m_);
            stop_ = true;
        }
        cv_.notify_all();
        for (auto& t : th_) t.join();
    }
    void start(std::function<void(int, int)> f) {
        wait();
        std::lock_guard<std::mutex> g(m_);
        job_ = std::move(f);
        pending_ = n_;
        ++gen_;
        cv_.notify_all();
    }
    void wait() {
        std::unique_lock<std::mutex> g(m_);
        done_.wait(g, [this] { return pending_ == 0; });
    }

private:
    void loop(int w) {
        uint64_t seen = 0;
        for (;;) {
            std::function<void(int, int)> f;
            {
                std::unique_lock<std::mutex> g(m_);
                cv_.wait(g, [&] { return stop_ || gen_ != seen; });
                if (stop_) return;
                seen = gen_;
                f = job_;
            }
            f(w, n_);
            std::lock_guard<std::mutex> g(m_);
            if (--pending_ == 0) done_.notify_all();
        }
    }
    int n_;
    std::vector<std::thread> th_;
    std::mutex m_;
    std::condition_variable cv_, done_;
    std::function<void(int, int)> job_;
    uint64_t gen_ = 0;
    int pending_ = 0;
    bool stop_ = false;
};
}  // namespace

// Delta merge staged by hetm_dev_merge_prepare before the round's verdict.
struct PreparedMerge {
    bool active = false;
    bool speculative = false;  // the records were swapped into `host` already
    uint64_t n_slots = 0;      // write-set log slots of the round when staged
    uint64_t n_rec = 0, k0 = 0, pieces = 0;  // delta records, first DMA'd piece, pieces
    uint64_t round_tx = 0;     // the round's submitted transactions when staged
    uint64_t* host = nullptr;
    int buf = 0;               // delta buffer holding it
};

struct hetm_dev {
    hetm_dev_config cfg{};
    int device = 0;
    uint64_t W = 0, base = 0;
    uint32_t gran_shift = 0, chunk_shift = 0;
    uint64_t rs_bits = 0, rs_words = 0, chunk_bits = 0, chunk_words = 0;
    uint32_t max_attempts = 1u << 24;

    Cell* d_cells = nullptr;             // devReplica: {value, lock, ts, spare} per word
    uint64_t* d_shadow = nullptr;        // devShadow: plain words
    uint64_t* d_stage = nullptr;         // plain-word staging for raw ops / basic rollback
    uint64_t stage_cap = 0;
    unsigned long long* d_rs = nullptr;
    unsigned long long* d_ws = nullptr;
    unsigned long long* d_chunk = nullptr;
    DevCounters* d_ctr = nullptr;
    DevCounters* h_ctr = nullptr;        // pinned mirror of d_ctr
    uint64_t* h_first = nullptr;         // pinned: first ticket of the current host-buffer batch
    unsigned long long* d_pop = nullptr; // popcount scratch (3)
    unsigned long long* d_restore = nullptr; // apply-kernel restore queue (restore_cap entries)
    uint64_t restore_cap = 0;
    CacheGeom cache{};                   // HETM_KERNEL_CACHE region
    hetm_cache_result* d_res = nullptr;  // per-transaction results (host-buffer path)
    uint64_t res_cap = 0;
    uint32_t* d_wlog = nullptr;          // write-set log (2 slots per commit ticket of the round)
    uint64_t wlog_slots = 0;
    uint64_t round_tx = 0;               // transactions submitted this round (ticket upper bound)
    DeltaScratch ds{};                   // delta claim bitmap / unique words / bucket counts (cells.cu)
    uint64_t* h_nrec = nullptr;          // pinned: record count of the last staged delta
    cudaEvent_t ev_nrec = nullptr;       // ... landed in h_nrec
    cudaEvent_t ev_pick = nullptr;       // merge_stage: the pick/claim pass is done (s_merge)
    // hetm_dev_merge_stage: the round's delta staged in HBM + devShadow refreshed
    // (the device half of mergeCommit), not yet shipped to the host
    struct {
        bool active = false;
        uint64_t round_tx = 0;
        int buf = 0;
    } staged;
    // merge delta (device) and its pinned host landing buffer, double-buffered:
    // a round's delta is staged while the worker pool still scatters the
    // previous round's (hetm_dev_merge_prepare)
    DeltaBuf d_delta[2] = {{nullptr, nullptr}, {nullptr, nullptr}};
    DeltaBuf h_delta[2] = {{nullptr, nullptr}, {nullptr, nullptr}};
    uint64_t delta_cap = 0;
    std::vector<cudaEvent_t> piece_ev[2];  // per-piece D2H completion of each buffer
    int dbuf = 0;                          // the buffer the next delta is staged into
    std::unique_ptr<WorkerPool> pool;    // host scatter of the delta into host_replica
    hetm_log_entry* d_arena = nullptr;   // this round's host log, in arrival order
    uint64_t arena_cap = 0, arena_n = 0;
    std::vector<std::pair<uint64_t, uint64_t>> deferred;  // [lo,hi) streamed VALIDATE_ONLY, not applied
    bool deferred_final = false;         // deferred ranges re-validated after execution ended
    // early-validation cadence: VALIDATE_ONLY chunks are validated
    // in one launch every ev_period chunks; arena [ev_lo, arena_n) is pending
    uint32_t ev_period = 8;
    uint32_t ev_pending = 0;
    uint64_t ev_lo = 0;
    // per-chunk delivery handles (bus.hpp:51-56 Delivery): handle h's H2D copy
    // is complete when dl_ev[h % kDeliveryRing] has fired; handles below
    // dl_floor are known complete (s_copy is in order)
    std::vector<cudaEvent_t> dl_ev;
    uint64_t dl_next = 0, dl_floor = 0;
    std::map<int, hetm_source_stats> sources;  // per source thread, this round
    uint32_t recv_applied = 0;  // bit p: the peer-arena regions of parity p were applied this round
    bool merge_staged = false;  // hetm_dev_merge_stage ran this round: no more batches / chunks
    // every batch of the round committed with per-word versions (bank / rw
    // kernels): the delta merge picks words by version instead of claiming them
    bool round_versioned = true;
    void* d_in = nullptr;
    uint64_t in_cap = 0;
    unsigned long long* d_tk = nullptr;
    uint64_t tk_cap = 0;
    void* d_route = nullptr;
    size_t route_cap = 0;
    // peer delivery (route_to_peers): this shard's receive arena + bucket counts
    hetm_log_entry* d_recv = nullptr;
    unsigned long long* d_recv_counts = nullptr;
    uint32_t recv_shards = 0;
    uint64_t recv_cap = 0;
    void** d_peer_ptrs = nullptr;  // device copy of {entries[64], counts[64]} peer pointer tables, per parity
    std::array<void*, 128> peer_table[2];  // host copies of the uploaded tables
    bool peer_table_ok[2] = {false, false};
    unsigned long long* d_peer_totals = nullptr;
    void* d_flush = nullptr;
    size_t flush_bytes = 0;
    unsigned flush_gen = 0;

    cudaStream_t s_exec = nullptr, s_copy = nullptr, s_val = nullptr, s_merge = nullptr, s_d2h = nullptr,
                 s_zc = nullptr,  // s_zc: zero-copy delta stores into the host replica
        s_in = nullptr, s_out = nullptr;  // pipelined host-input batches: input pieces in, tickets/results out
    unsigned long long* d_trace = nullptr;  // checker trace of the armed batch (kTraceWords per tx)
    uint64_t trace_cap = 0;                 // in transactions
    uint64_t* trace_out = nullptr;          // armed by hetm_dev_trace_next_batch
    uint32_t fault = 0;                     // HETM_FAULT_* (checker mutation suite)
    int schedule = HETM_SCHED_AUTO;         // bank batch schedule (hetm_dev_set_schedule)
    uint32_t auto_scan_left = 0;            // AUTO feedback: device-pointer bank batches still to run as SCAN
    uint32_t apply_amax_left = 0;           // apply launches still to run in the atomicMax form (hot logs)
    uint64_t applied_since_read = 0;        // log entries applied since the counters were last read
    unsigned long long last_apply_dups = 0; // DevCounters::apply_dups at that read
    uint64_t dptr_feedback_n = 0;           // last batch: an optimistic AUTO device-pointer bank batch of n tx
    uint32_t* h_hot = nullptr;              // device-side hot-spot estimate (mapped host word)
    uint32_t* d_hot = nullptr;
    cudaStream_t s_est = nullptr;           // the estimator runs off the batch's critical path
    cudaEvent_t ev_est = nullptr;
    hetm_bank_tx* d_est_in = nullptr;       // the estimate's copy of the sampled input records
    void* d_sched = nullptr;                // SCAN schedule scratch (bank_sched_temp_bytes)
    size_t sched_bytes = 0;
    SchedGraph sched_graph;                 // its captured launch sequence
    PreparedMerge prep;                     // hetm_dev_merge_prepare state
    cudaEvent_t ev_stage = nullptr;         // delta records gathered (s_merge)
    // merge_stage: the devShadow patch with the host-log winners runs on s_win
    // beside the pick/emit on s_merge (disjoint words in a committed round)
    cudaStream_t s_win = nullptr;
    cudaEvent_t ev_win_fork = nullptr, ev_win = nullptr;
    bool win_side = false;
    unsigned long long* d_rs_zero = nullptr;  // all-zero RS bitmap (HETM_FAULT_SKIP_RS)
    unsigned int* d_stripes = nullptr;        // bank kernel lock-stripe table (phased_tx.cuh KO_STRIPES)
    uint32_t stripe_shift = 64;
    std::vector<cudaEvent_t> in_ev;       // per-piece input H2D landed
    std::vector<cudaEvent_t> kp_ev;       // per-piece kernel start/end (timing events)
    cudaEvent_t ev_exec = nullptr, ev_copy = nullptr, ev_val = nullptr, ev_round = nullptr, ev_shadow = nullptr,
                ev_d2h = nullptr, ev_t0 = nullptr, ev_t1 = nullptr, ev_copy_zc = nullptr,
                ev_ext = nullptr;
    bool intake_open = true;
    bool shadow_synced = true;   // devShadow == devReplica as of the round start
    bool round_applied = false;  // some APPLY validation touched devReplica this round
    bool d2h_pending = false;
    std::set<int> kernels;
    std::vector<hetm_transfer_record> xfer;
    std::mutex mu;
    std::string last_err;
    LaunchGeom geom{};
    uint64_t bytes_alloc = 0;
    uint64_t l2_bytes = 0;
    hetm_batch_stats last_batch{};
    bool timing = false;
    std::vector<std::pair<cudaEvent_t, cudaEvent_t>> tpairs[3];  // recorded launch brackets: batch, validation, merge stage
    std::vector<cudaEvent_t> tpool;

    cudaEvent_t tev() {
        if (!tpool.empty()) {
            cudaEvent_t e = tpool.back();
            tpool.pop_back();
            return e;
        }
        cudaEvent_t e = nullptr;
        cudaEventCreate(&e);
        return e;
    }

    ShardView view() const {
        ShardView v;
        v.cells = d_cells;
        v.base = base;
        v.size_words = W;
        v.rs = d_rs;
        v.ws = d_ws;
        v.chunk = d_chunk;
        v.gran_shift = gran_shift;
        v.chunk_shift = chunk_shift;
        v.wlog = d_wlog;
        v.wlog_slots = wlog_slots;
        v.wlog_ovf = &d_ctr->wlog_overflow;
        v.serial = (cfg.flags & HETM_CFG_DETERMINISTIC) ? 1u : 0u;
        v.trace = nullptr;
        v.stripes = d_stripes;
        v.stripe_shift = stripe_shift;
        return v;
    }
    std::mutex xfer_mu;  // record() is reached from the GPU-controller and the log streamer threads
    void record(int dir, int tag, uint64_t bytes) {
        std::lock_guard<std::mutex> g(xfer_mu);
        xfer.push_back(hetm_transfer_record{dir, tag, bytes});
    }
};

namespace {

int fail(hetm_dev* d, cudaError_t e, const char* what) {
    if (d) {
        d->last_err = std::string(what) + ": " + cudaGetErrorString(e);
    }
    std::fprintf(stderr, "[hetm_b200] CUDA error in %s: %s\n", what, cudaGetErrorString(e));
    return HETM_ERR_CUDA;
}

#define CK(dev, x)                                         \
    do {                                                   \
        cudaError_t e_ = (x);                              \
        if (e_ != cudaSuccess) return fail(dev, e_, #x);   \
    } while (0)

bool pow2(uint64_t v) { return v && !(v & (v - 1)); }
uint32_t log2u(uint64_t v) { return (uint32_t)__builtin_ctzll(v); }

int sync_all(hetm_dev* d);

int dev_alloc(hetm_dev* d, void** p, size_t bytes) {
    cudaError_t e = cudaMalloc(p, bytes ? bytes : 16);
    if (e != cudaSuccess) return fail(d, e, "cudaMalloc");
    d->bytes_alloc += bytes;
    return HETM_OK;
}

int ensure_stage(hetm_dev* d, uint64_t words) {
    if (words <= d->stage_cap) return HETM_OK;
    if (d->d_stage) {
        int rc = sync_all(d);
        if (rc) return rc;
        cudaFree(d->d_stage);
        d->bytes_alloc -= d->stage_cap * 8;
    }
    d->stage_cap = std::max<uint64_t>(words, 1 << 16);
    return dev_alloc(d, (void**)&d->d_stage, d->stage_cap * 8);
}

int check_range(hetm_dev* d, uint64_t addr, uint64_t n) {
    if (addr < d->base) return HETM_ERR_OUT_OF_BOUNDS;
    const uint64_t loc = addr - d->base;
    if (loc >= d->W || n > d->W - loc) return HETM_ERR_OUT_OF_BOUNDS;
    return HETM_OK;
}

int sync_all(hetm_dev* d) {
    CK(d, cudaStreamSynchronize(d->s_exec));
    CK(d, cudaStreamSynchronize(d->s_copy));
    CK(d, cudaStreamSynchronize(d->s_val));
    CK(d, cudaStreamSynchronize(d->s_merge));
    CK(d, cudaStreamSynchronize(d->s_d2h));
    if (d->s_est) CK(d, cudaStreamSynchronize(d->s_est));
    return HETM_OK;
}

constexpr uint64_t kDeliveryRing = 4096;  // delivery events in flight per handle

constexpr uint64_t kApplyHotRatio = 64;   // apply: put-backs per applied entry above 1/64 ...
constexpr uint32_t kApplyAmaxRun = 16;     // ... run the next 16 apply launches in the atomicMax form
constexpr uint64_t kAutoRetryRatio = 1024; // AUTO feedback: transactions needing a 3rd attempt above 1/1024
                                           // (stripe kernel: uniform 0.035 %, zipf 0.4 0.046 %, zipf 0.5
                                           // 0.23 %, profiles/r02z_skew.txt) ...
constexpr uint32_t kAutoScanRun = 15;      // ... run the next 15 bank batches as SCAN

int read_counters(hetm_dev* d) {
    CK(d, cudaMemcpy(d->h_ctr, d->d_ctr, sizeof(DevCounters), cudaMemcpyDeviceToHost));
    // AUTO feedback for device-pointer batches, judged when the caller syncs the
    // counters (verdict, stats): an optimistic bank batch in which more than 1
    // transaction per 1024 needed a third attempt had conflict chains the sample
    // did not predict (the zipf ~0.5 band, where SCAN wins 2x: 0.31 vs 0.62-0.67
    // ms).  Repeated aborts of ONE transaction, not the abort count: stripe false
    // sharing aborts 1.8 % of uniform transfers once but almost never twice
    // (profiles/r02z_skew.txt).  The next kAutoScanRun device-pointer batches run
    // as SCAN, then the optimistic kernel is tried again.
    if (d->dptr_feedback_n) {
        if (d->h_ctr->retried * kAutoRetryRatio > d->dptr_feedback_n) d->auto_scan_left = kAutoScanRun;
        d->dptr_feedback_n = 0;
    }
    // apply form feedback (validate.cu apply_xchg_kernel): the exchange form's
    // put-backs count the log's repeated words; a hot log (zipf, configs[2])
    // runs the next kApplyAmaxRun launches in the atomicMax form
    const unsigned long long dups = d->h_ctr->apply_dups - d->last_apply_dups;
    d->last_apply_dups = d->h_ctr->apply_dups;
    if (d->applied_since_read && dups * kApplyHotRatio > d->applied_since_read) d->apply_amax_left = kApplyAmaxRun;
    d->applied_since_read = 0;
    return HETM_OK;
}

// Restore queue + apply form of the next apply launch over n entries.
RestoreQueue apply_queue(hetm_dev* d, uint64_t n) {
    RestoreQueue rq{d->d_restore, d->restore_cap};
    if (d->apply_amax_left) {
        rq.amax = 1;
        --d->apply_amax_left;
    }
    d->applied_since_read += n;
    return rq;
}

size_t record_bytes(int kernel_id) {
    switch (kernel_id) {
        case HETM_KERNEL_BANK: return sizeof(hetm_bank_tx);
        case HETM_KERNEL_RW: return sizeof(hetm_rw_tx);
        case HETM_KERNEL_CACHE: return sizeof(hetm_cache_tx);
        default: return 0;
    }
}

// Grow the write-set log to hold 2 slots per transaction submitted this round
// (+ n more).  Shards of >= 2^32 words keep it disabled (chunk merge only).
int ensure_wlog(hetm_dev* d, uint64_t n) {
    if (d->W >= (1ull << 32)) return HETM_OK;
    // tickets of attempts that aborted after taking one also own slots: +25% headroom
    // (a round that outruns it merges by chunks; the log is only an accelerator)
    const uint64_t need = 2 * (d->round_tx + n) + (d->round_tx + n) / 2 + 65536;
    if (need <= d->wlog_slots) return HETM_OK;
    const uint64_t cap = std::max<uint64_t>({need, 2 * d->wlog_slots, 1ull << 21});
    int rc = sync_all(d);
    if (rc) return rc;
    void* p = nullptr;
    if ((rc = dev_alloc(d, &p, cap * 4))) return rc;
    if (d->d_wlog) {
        // the round's slots in use: 2 per ticket taken since the round's origin
        // (aborted attempts that took a ticket own slots too, so this can exceed
        // 2 * round_tx); a span past the old capacity lost slots the kernels
        // could not store, which the kernels flagged as an overflow already
        unsigned long long tk[2] = {0, 0};  // {ticket, wlog_base}
        CK(d, cudaMemcpy(&tk[0], &d->d_ctr->ticket, 8, cudaMemcpyDeviceToHost));
        CK(d, cudaMemcpy(&tk[1], &d->d_ctr->wlog_base, 8, cudaMemcpyDeviceToHost));
        const uint64_t span = 2 * (tk[0] - tk[1]);
        const uint64_t used = std::min<uint64_t>(span, d->wlog_slots);
        if (used) CK(d, cudaMemcpy(p, d->d_wlog, used * 4, cudaMemcpyDeviceToDevice));
        if (span > d->wlog_slots) {
            const unsigned long long one = 1;
            CK(d, cudaMemcpy(&d->d_ctr->wlog_overflow, &one, 8, cudaMemcpyHostToDevice));
        }
        cudaFree(d->d_wlog);
        d->bytes_alloc -= d->wlog_slots * 4;
    }
    d->d_wlog = static_cast<uint32_t*>(p);
    d->wlog_slots = cap;
    return HETM_OK;
}

// Enqueue one batch kernel on `s` (inputs and tickets are device pointers).
// Hot-spot estimate of a host-resident bank batch (HETM_SCHED_AUTO): the
// access count of the hottest account among 4096 sampled transactions, scaled
// to the batch, estimates the longest chain of conflicting commits the
// optimistic kernel would serialize (~1.4 us per link on B200,
// profiles/r01_sched_crossover.txt); from 768 (HETM_SCHED_CHAIN) the SCAN
// schedule wins.
uint64_t sched_chain() {
    static const uint64_t chain = [] {
        const char* e = std::getenv("HETM_SCHED_CHAIN");
        return e ? std::strtoull(e, nullptr, 10) : 768ull;
    }();
    return chain;
}
// A count of >= 3 in the sample is required: chance pairs are common under
// uniform access (8 K sampled accounts over 2^26 meet ~0.5 times).
bool hot_chain(uint64_t best, uint64_t n, uint64_t S, uint64_t chain) { return best >= 3 && best * n / S >= chain; }

bool bank_batch_hot(const hetm_bank_tx* in, uint64_t n) {
    const uint64_t chain = sched_chain();
    constexpr uint64_t kBlocks = 32, kPerBlock = 128, kSlots = 1 << 15;
    if (n * 4 < chain) return false;
    // 32 evenly spaced blocks of 128 consecutive transactions: the reads stream
    // (the worker pool may be saturating host DRAM with the previous merge —
    // 4096 scattered cache misses cost ~0.4 ms then, 32 cost nothing); the
    // per-thread table is reused across batches (a generation tag replaces the clear)
    const uint64_t per = std::min<uint64_t>(kPerBlock, n / kBlocks ? n / kBlocks : 1);
    const uint64_t nb = n < kBlocks ? n : kBlocks, S = nb * per;
    thread_local std::vector<uint32_t> key(kSlots), cnt(kSlots), tag(kSlots);
    thread_local uint32_t gen = 0;
    if (++gen == 0) {
        std::fill(tag.begin(), tag.end(), 0u);
        gen = 1;
    }
    uint32_t best = 0;
    for (uint64_t blk = 0; blk < nb; ++blk) {
        const hetm_bank_tx* b = in + blk * (n / nb);
        for (uint64_t q = 0; q < per; ++q)
            for (uint32_t a : b[q].acct) {
                uint64_t h = (a * 0x9e3779b97f4a7c15ull) >> 49;  // 15 bits
                while (tag[h] == gen && key[h] != a) h = (h + 1) & (kSlots - 1);
                if (tag[h] != gen) {
                    tag[h] = gen;
                    key[h] = a;
                    cnt[h] = 0;
                }
                best = std::max(best, ++cnt[h]);
            }
    }
    return hot_chain(best, n, S, chain);
}

// AUTO runs cache batches of at least this size as SCAN: it is faster at any
// skew (one set per thread, no set-lock handoffs; 0.48 vs 0.97 ms per 2^20
// GET/SET 90/10, profiles/r01_configs_probe.json), while tiny batches do not
// amortize its sort.
constexpr uint64_t kCacheScanMin = 1u << 13;

int ensure_sched(hetm_dev* d, uint64_t n, int kernel_id = HETM_KERNEL_BANK) {
    const size_t need = kernel_id == HETM_KERNEL_CACHE ? cache_sched_temp_bytes(n, d->cache.n_sets)
                                                       : bank_sched_temp_bytes(n, d->W);
    if (need <= d->sched_bytes) return HETM_OK;
    if (d->d_sched) {
        CK(d, cudaDeviceSynchronize());
        cudaFree(d->d_sched);
        d->bytes_alloc -= d->sched_bytes;
        d->d_sched = nullptr;
        d->sched_bytes = 0;
    }
    if (int rc = dev_alloc(d, &d->d_sched, need)) return rc;
    d->sched_bytes = need;
    return HETM_OK;
}

extern "C" void cancel_prepare(hetm_dev* d);  // defined with the merge code (C linkage block)

int enqueue_batch(hetm_dev* d, int kernel_id, const void* d_inputs, uint64_t n, unsigned long long* d_tickets,
                  void* d_results, cudaStream_t s, bool reset_counters = true, unsigned long long* trace = nullptr,
                  bool hot = false) {
    if (d->merge_staged) return HETM_ERR_STATE;  // the round's merge has started (hetm_dev_merge_stage)
    cancel_prepare(d);  // a new batch of the round: a staged merge would miss it
    if (int rc = ensure_wlog(d, n)) return rc;
    if (kernel_id == HETM_KERNEL_CACHE) d->round_versioned = false;  // set-granular locks: claim the words
    CK(d, cudaStreamWaitEvent(s, d->ev_round, 0));
    CK(d, cudaStreamWaitEvent(s, d->ev_shadow, 0));  // shadow refresh reads devReplica
    if (reset_counters)  // committed, aborts, livelocked, retried: adjacent, one memset
        CK(d, cudaMemsetAsync(&d->d_ctr->committed, 0, 4 * sizeof(unsigned long long), s));
    cudaError_t e = cudaSuccess;
    cudaEvent_t t0 = nullptr, t1 = nullptr;
    if (d->timing) {
        t0 = d->tev();
        t1 = d->tev();
        CK(d, cudaEventRecord(t0, s));
    }
    ShardView v = d->view();
    v.trace = trace;
    // bank: SCAN schedule in the deterministic mode (same input order, no
    // single worker), when requested, or under AUTO for a hot batch
    const bool scan = kernel_id == HETM_KERNEL_BANK &&
                      (v.serial || d->schedule == HETM_SCHED_SCAN || (d->schedule == HETM_SCHED_AUTO && hot));
    if (scan) {
        if (int rc = ensure_sched(d, n)) return rc;
        static const bool use_graph = [] {  // HETM_SCHED_GRAPH=0: launch kernel by kernel (experiments)
            const char* e = std::getenv("HETM_SCHED_GRAPH");
            return !e || std::atoi(e) != 0;
        }();
        e = launch_bank_sched(v, static_cast<const hetm_bank_tx*>(d_inputs), n, d_tickets, d->d_ctr, d->d_sched,
                              d->sched_bytes, d->geom, s, use_graph ? &d->sched_graph : nullptr);
    } else if (kernel_id == HETM_KERNEL_CACHE &&
               (v.serial || d->schedule == HETM_SCHED_SCAN || (d->schedule == HETM_SCHED_AUTO && n >= kCacheScanMin))) {
        if (int rc = ensure_sched(d, n, kernel_id)) return rc;
        e = launch_cache_sched(v, d->cache, static_cast<const hetm_cache_tx*>(d_inputs), n, d_tickets,
                               static_cast<hetm_cache_result*>(d_results), d->d_ctr, d->d_sched, d->sched_bytes,
                               d->geom, s);
    } else if (kernel_id == HETM_KERNEL_BANK)
        e = launch_bank_batch(v, static_cast<const hetm_bank_tx*>(d_inputs), n, d_tickets, d->d_ctr,
                              d->max_attempts, d->geom, s);
    else if (kernel_id == HETM_KERNEL_CACHE)
        e = launch_cache_batch(d->view(), d->cache, static_cast<const hetm_cache_tx*>(d_inputs), n, d_tickets,
                               static_cast<hetm_cache_result*>(d_results), d->d_ctr, d->max_attempts, d->geom, s);
    else
        e = launch_rw_batch(v, static_cast<const hetm_rw_tx*>(d_inputs), n, d_tickets, d->d_ctr,
                            d->max_attempts, d->geom, s);
    if (e != cudaSuccess) return fail(d, e, "batch kernel launch");
    if (d->timing) {
        CK(d, cudaEventRecord(t1, s));
        d->tpairs[0].emplace_back(t0, t1);
    }
    CK(d, cudaEventRecord(d->ev_exec, s));
    d->round_tx += n;
    return HETM_OK;
}

// The apply restore queue holds a quarter of the largest apply launch (at
// least kRestoreCap): at cfg5 sizes (2^26 entries into a 2^31-word shard) ~2^20
// entries race with an earlier entry of the round, and an overflow costs a
// full winner pass over the launch.  Growing waits for the launches using it.
int ensure_restore(hetm_dev* d, uint64_t n) {
    const uint64_t need = std::max<uint64_t>(kRestoreCap, n / 4);
    if (need <= d->restore_cap) return HETM_OK;
    if (int rc = sync_all(d)) return rc;
    cudaFree(d->d_restore);
    d->bytes_alloc -= d->restore_cap * 8;
    d->d_restore = nullptr;
    d->restore_cap = 0;
    if (int rc = dev_alloc(d, (void**)&d->d_restore, need * 8)) return rc;
    d->restore_cap = need;
    return HETM_OK;
}

// Validation launch with optional timing brackets.
cudaError_t timed_validate(hetm_dev* d, const hetm_log_entry* log, uint64_t n, int apply, cudaStream_t s) {
    cudaEvent_t t0 = nullptr, t1 = nullptr;
    if (d->timing && n) {
        t0 = d->tev();
        t1 = d->tev();
        cudaEventRecord(t0, s);
    }
    ShardView v = d->view();
    if (d->fault & HETM_FAULT_SKIP_RS) v.rs = d->d_rs_zero;  // mutation: the RS test never fires
    cudaError_t e = (apply && (d->fault & HETM_FAULT_SKIP_TS))
                        ? launch_blind_apply(v, log, n, d->d_ctr, d->geom, s)  // mutation: no TS freshness
                        : launch_validate(v, log, n, apply, d->d_ctr, apply ? apply_queue(d, n) : RestoreQueue{d->d_restore, d->restore_cap},
                                          d->geom, s);
    if (d->timing && n) {
        cudaEventRecord(t1, s);
        d->tpairs[1].emplace_back(t0, t1);
    }
    return e;
}

int ensure_arena(hetm_dev* d, uint64_t need) {
    if (need <= d->arena_cap) return HETM_OK;
    uint64_t cap = std::max<uint64_t>(need, d->arena_cap * 2);
    int rc = sync_all(d);
    if (rc) return rc;
    void* p = nullptr;
    if ((rc = dev_alloc(d, &p, cap * sizeof(hetm_log_entry)))) return rc;
    if (d->arena_n) CK(d, cudaMemcpy(p, d->d_arena, d->arena_n * sizeof(hetm_log_entry), cudaMemcpyDeviceToDevice));
    cudaFree(d->d_arena);
    d->bytes_alloc -= d->arena_cap * sizeof(hetm_log_entry);
    d->d_arena = static_cast<hetm_log_entry*>(p);
    d->arena_cap = cap;
    return HETM_OK;
}

// The round's host log on this device: the arena plus the received peer
// regions applied this round (their counts stay on the device).
RoundLogs round_logs(hetm_dev* d) {
    RoundLogs l{};
    l.flat = d->d_arena;
    l.n = d->arena_n;
    for (uint32_t p = 0; p < 2; ++p)
        if (d->recv_applied & (1u << p))
            l.region[l.n_regions_sets++] = RoundLogRegions{d->d_recv + (uint64_t)p * d->recv_shards * d->recv_cap,
                                                           d->d_recv_counts + p * 64, d->recv_shards, d->recv_cap};
    return l;
}

// devShadow patch with the winners of the round's host log (the words the
// validation applied), on s_merge; gate: skipped on the device on a conflict.
cudaError_t patch_shadow(hetm_dev* d, const DevCounters* gate = nullptr, cudaStream_t s = nullptr) {
    const RoundLogs l = round_logs(d);
    if (!s) s = d->s_merge;
    cudaError_t e = launch_winner_apply(d->d_cells, d->d_shadow, d->base, d->W, l.flat, l.n, d->geom, s, gate);
    for (uint32_t k = 0; k < l.n_regions_sets && e == cudaSuccess; ++k)
        e = launch_winner_regions(d->d_cells, d->d_shadow, d->base, d->W, l.region[k].base, l.region[k].counts,
                                  l.region[k].n_regions, l.region[k].cap, d->geom, s, gate);
    return e;
}

// Dirty chunks of this round as coalesced [offset, bytes) word ranges
// (adjacent dirty chunks form one transfer descriptor).
int dirty_ranges(hetm_dev* d, std::vector<std::pair<uint64_t, uint64_t>>& out, uint64_t* n_dirty) {
    std::vector<uint64_t> bits(d->chunk_words);
    CK(d, cudaMemcpy(bits.data(), d->d_chunk, d->chunk_words * 8, cudaMemcpyDeviceToHost));
    const uint64_t wpc = 1ull << d->chunk_shift;
    uint64_t c = 0, nd = 0;
    out.clear();
    while (c < d->chunk_bits) {
        if (!((bits[c >> 6] >> (c & 63)) & 1ull)) {
            ++c;
            continue;
        }
        const uint64_t first = c;
        while (c < d->chunk_bits && ((bits[c >> 6] >> (c & 63)) & 1ull)) ++c;
        nd += c - first;
        const uint64_t lo = first * wpc, hi = std::min(c * wpc, d->W);
        out.emplace_back(lo, hi - lo);
    }
    *n_dirty = nd;
    return HETM_OK;
}

// devShadow := devReplica on s_merge.  Incremental when the shadow held the
// round-start state: device-dirty chunks are copied and the round's host log
// winners are patched in; otherwise a full D2D copy.
int refresh_shadow(hetm_dev* d, bool host_log_applied, uint64_t dirty_bytes) {
    if (!d->d_shadow) return HETM_OK;
    if (d->d2h_pending) CK(d, cudaStreamWaitEvent(d->s_merge, d->ev_d2h, 0));
    if (d->shadow_synced) {
        cudaError_t e = launch_dirty_chunks(d->d_shadow, d->d_cells, d->W, d->d_chunk, d->chunk_bits, d->chunk_shift,
                                            true, d->geom, d->s_merge);
        if (e != cudaSuccess) return fail(d, e, "dirty_chunks(shadow)");
        if (host_log_applied) {
            e = patch_shadow(d);
            if (e != cudaSuccess) return fail(d, e, "winner_apply(shadow)");
        }
        d->record(HETM_D2D, HETM_TAG_SHADOW, dirty_bytes);
    } else {
        cudaError_t e = launch_dirty_chunks(d->d_shadow, d->d_cells, d->W, nullptr, d->chunk_bits, d->chunk_shift, true,
                                            d->geom, d->s_merge);
        if (e != cudaSuccess) return fail(d, e, "dirty_chunks(full shadow)");
        d->record(HETM_D2D, HETM_TAG_SHADOW, d->W * 8);
        d->shadow_synced = true;
    }
    CK(d, cudaEventRecord(d->ev_shadow, d->s_merge));
    return HETM_OK;
}

int wait_round_work(hetm_dev* d, cudaStream_t s) {
    CK(d, cudaEventRecord(d->ev_val, d->s_val));
    CK(d, cudaStreamWaitEvent(s, d->ev_exec, 0));
    CK(d, cudaStreamWaitEvent(s, d->ev_val, 0));
    return HETM_OK;
}

// Round work enqueued on a caller's stream (validate_dptr, apply_received,
// bitmap_or_peers) joins the validation stream at once, so ev_val (recorded on
// s_val by wait_round_work) and the verdict's s_val sync cover it.
int join_val(hetm_dev* d, cudaStream_t s) {
    if (s == d->s_val) return HETM_OK;
    CK(d, cudaEventRecord(d->ev_ext, s));
    CK(d, cudaStreamWaitEvent(d->s_val, d->ev_ext, 0));
    return HETM_OK;
}

int enqueue_deferred_apply(hetm_dev* d) {
    if (d->deferred.empty()) return HETM_OK;
    CK(d, cudaStreamWaitEvent(d->s_val, d->ev_exec, 0));
    for (auto& r : d->deferred) {
        if (int rc = ensure_restore(d, r.second - r.first)) return rc;
        cudaError_t e = timed_validate(d, d->d_arena + r.first, r.second - r.first, 1, d->s_val);
        if (e != cudaSuccess) return fail(d, e, "validate(apply deferred)");
    }
    d->deferred.clear();
    d->deferred_final = false;
    d->round_applied = true;
    d->ev_lo = d->arena_n;  // the apply launches validated the pending early chunks too
    d->ev_pending = 0;
    return HETM_OK;
}

}  // namespace

extern "C" {

const char* hetm_strerror(int s) {
    switch (s) {
        case HETM_OK: return "ok";
        case HETM_ERR_INVALID_SIZE: return "invalid-size";
        case HETM_ERR_OUT_OF_BOUNDS: return "out-of-bounds";
        case HETM_ERR_ROUND_CLOSED: return "round-closed";
        case HETM_ERR_KERNEL_NOT_REGISTERED: return "kernel-not-registered";
        case HETM_ERR_LIVELOCK: return "livelock-budget-exceeded";
        case HETM_ERR_NO_IMPLEMENTATION: return "no-implementation";
        case HETM_ERR_BAD_AFFINITY: return "bad-affinity";
        case HETM_ERR_INCOMPLETE_TRACE: return "incomplete-trace";
        case HETM_ERR_NONDETERMINISTIC: return "nondeterministic-input";
        case HETM_ERR_CONFIG: return "config-invalid";
        case HETM_ERR_IO: return "io-error";
        case HETM_ERR_INVALID_ARG: return "invalid-argument";
        case HETM_ERR_CUDA: return "cuda-error";
        case HETM_ERR_NO_DEVICE: return "no-cuda-device";
        case HETM_ERR_NONMONOTONE_TS: return "non-monotone-timestamp";
        case HETM_ERR_STATE: return "invalid-round-state";
        default: return "unknown";
    }
}

int hetm_abi_version(void) { return HETM_B200_ABI_VERSION; }

int hetm_device_count(int* n) {
    if (!n) return HETM_ERR_INVALID_ARG;
    int c = 0;
    if (cudaGetDeviceCount(&c) != cudaSuccess) {
        cudaGetLastError();
        *n = 0;
        return HETM_ERR_NO_DEVICE;
    }
    *n = c;
    return c > 0 ? HETM_OK : HETM_ERR_NO_DEVICE;
}

void hetm_dev_config_default(hetm_dev_config* c) {
    if (!c) return;
    std::memset(c, 0, sizeof(*c));
    c->rs_gran_bytes = 1024;   // SPEC.md:239 default
    c->chunk_bytes = 16384;    // bitmap.hpp:130
}

int hetm_dev_open(const hetm_dev_config* cfg, hetm_dev** out) {
    if (!cfg || !out) return HETM_ERR_INVALID_ARG;
    *out = nullptr;
    // stmr.create pre-conditions, bitmap geometry (bitmap.hpp:99-100,134-135)
    if (cfg->size_words == 0) return HETM_ERR_INVALID_SIZE;
    if (!pow2(cfg->rs_gran_bytes) || cfg->rs_gran_bytes % 8) return HETM_ERR_INVALID_SIZE;
    if (!pow2(cfg->chunk_bytes) || cfg->chunk_bytes % 8) return HETM_ERR_INVALID_SIZE;
    const uint64_t align_words = std::max(cfg->rs_gran_bytes, cfg->chunk_bytes) / 8;
    if (cfg->shard_base % align_words) return HETM_ERR_CONFIG;
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
        cudaGetLastError();
        return HETM_ERR_NO_DEVICE;
    }
    if (cfg->device < 0 || cfg->device >= ndev) return HETM_ERR_CONFIG;

    hetm_dev* d = new hetm_dev();
    d->cfg = *cfg;
    d->device = cfg->device;
    d->W = cfg->size_words;
    d->base = cfg->shard_base;
    d->cache.base_local = 0;  // default cache region: the largest power-of-two set count that fits
    d->cache.n_sets = 2;
    while (d->cache.n_sets * 2 * HETM_CACHE_SET_WORDS <= d->W) d->cache.n_sets *= 2;
    d->gran_shift = log2u(cfg->rs_gran_bytes / 8);
    d->chunk_shift = log2u(cfg->chunk_bytes / 8);
    d->rs_bits = (d->W * 8 + cfg->rs_gran_bytes - 1) / cfg->rs_gran_bytes;  // bitmap.hpp:96-97 ceil
    d->rs_words = (d->rs_bits + 63) / 64;
    d->chunk_bits = (d->W * 8 + cfg->chunk_bytes - 1) / cfg->chunk_bytes;
    d->chunk_words = (d->chunk_bits + 63) / 64;
    if (cfg->max_attempts) d->max_attempts = cfg->max_attempts;

    auto bail = [&](int rc) {
        hetm_dev_close(d);
        return rc;
    };
    if (cudaSetDevice(d->device) != cudaSuccess) return bail(fail(d, cudaGetLastError(), "cudaSetDevice"));
    if (cfg->flags & HETM_CFG_L2_FETCH_32) cudaDeviceSetLimit(cudaLimitMaxL2FetchGranularity, 32);
    int rc;
    if ((rc = dev_alloc(d, (void**)&d->d_cells, d->W * sizeof(Cell)))) return bail(rc);
    if (!(cfg->flags & HETM_CFG_NO_SHADOW))
        if ((rc = dev_alloc(d, (void**)&d->d_shadow, d->W * 8))) return bail(rc);
    if ((rc = dev_alloc(d, (void**)&d->d_rs, d->rs_words * 8))) return bail(rc);
    if ((rc = dev_alloc(d, (void**)&d->d_ws, d->rs_words * 8))) return bail(rc);
    if ((rc = dev_alloc(d, (void**)&d->d_chunk, d->chunk_words * 8))) return bail(rc);
    if ((rc = dev_alloc(d, (void**)&d->d_ctr, sizeof(DevCounters)))) return bail(rc);
    {  // lock-stripe table of the bank kernel: 2^24 32-bit words (64 MiB: false-sharing aborts 1.8 % of
       // uniform transfers vs 6.6 % at 2^22, same batch time, profiles/r02x_stripe_skew.txt), fewer for
       // small shards
        static const uint32_t max_bits = [] {  // tuning experiments: HETM_STRIPE_BITS
            const char* e = std::getenv("HETM_STRIPE_BITS");
            return e ? (uint32_t)std::atoi(e) : 24u;
        }();
        uint32_t bits = 10;
        while (bits < max_bits && (1ull << bits) < d->W) ++bits;
        if ((rc = dev_alloc(d, (void**)&d->d_stripes, (4ull << bits)))) return bail(rc);
        d->stripe_shift = 64 - bits;
        CK(d, cudaMemset(d->d_stripes, 0, 4ull << bits));  // unlocked, version 0
    }
    {
        // Off by default: on s_win the merge stage drops 0.275 -> 0.258 ms, but the
        // next bank batch runs ~8 us slower (the emit's dirty lines are the last
        // ones left in L2 and drain under it), so the step gains only ~1 %
        // (profiles/r02au_winner_side_stream_ab.txt).  HETM_WIN_SIDE=1 turns it on.
        static const bool win_side = [] {
            const char* e = std::getenv("HETM_WIN_SIDE");
            return e && std::atoi(e) != 0;
        }();
        d->win_side = win_side;
    }
    if ((rc = dev_alloc(d, (void**)&d->d_pop, 4 * sizeof(unsigned long long)))) return bail(rc);
    if ((rc = dev_alloc(d, (void**)&d->d_restore, kRestoreCap * sizeof(unsigned long long)))) return bail(rc);
    d->restore_cap = kRestoreCap;
    d->arena_cap = cfg->log_capacity ? cfg->log_capacity : (1ull << 20);
    if ((rc = dev_alloc(d, (void**)&d->d_arena, d->arena_cap * sizeof(hetm_log_entry)))) return bail(rc);
    if (cudaHostAlloc((void**)&d->h_first, 64, cudaHostAllocPortable) != cudaSuccess)
        return bail(fail(d, cudaGetLastError(), "cudaHostAlloc(first ticket)"));
    if (cudaHostAlloc((void**)&d->h_ctr, sizeof(DevCounters), cudaHostAllocPortable) != cudaSuccess)
        return bail(fail(d, cudaGetLastError(), "cudaHostAlloc(counters)"));
    std::memset(d->h_ctr, 0, sizeof(DevCounters));

    // Stmr.create: all replicas zero-filled; locks/TS/bitmaps zero.
    CK(d, cudaMemset(d->d_cells, 0, d->W * sizeof(Cell)));
    if (d->d_shadow) CK(d, cudaMemset(d->d_shadow, 0, d->W * 8));
    CK(d, cudaMemset(d->d_rs, 0, d->rs_words * 8));
    CK(d, cudaMemset(d->d_ws, 0, d->rs_words * 8));
    CK(d, cudaMemset(d->d_chunk, 0, d->chunk_words * 8));
    CK(d, cudaMemset(d->d_ctr, 0, sizeof(DevCounters)));

    for (cudaStream_t* s : {&d->s_exec, &d->s_copy, &d->s_val, &d->s_merge, &d->s_d2h, &d->s_zc, &d->s_in, &d->s_out, &d->s_win})
        CK(d, cudaStreamCreateWithFlags(s, cudaStreamNonBlocking));
    for (cudaEvent_t* e : {&d->ev_exec, &d->ev_copy, &d->ev_val, &d->ev_round, &d->ev_shadow, &d->ev_d2h, &d->ev_copy_zc, &d->ev_stage, &d->ev_ext, &d->ev_win_fork, &d->ev_win})
        CK(d, cudaEventCreateWithFlags(e, cudaEventDisableTiming));
    CK(d, cudaEventCreate(&d->ev_t0));
    CK(d, cudaEventCreate(&d->ev_t1));
    // Record the "round boundary" events once so the first waits are satisfied.
    CK(d, cudaEventRecord(d->ev_round, d->s_merge));
    CK(d, cudaEventRecord(d->ev_exec, d->s_exec));
    CK(d, cudaEventRecord(d->ev_d2h, d->s_d2h));

    int sms = 0;
    CK(d, cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, d->device));
    int l2 = 0;
    CK(d, cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, d->device));
    d->l2_bytes = (uint64_t)l2;
    d->geom.sm_count = sms;
    int b = 0;
    // Batch kernels: ONE resident 256-thread CTA per SM.  The bank batch is
    // bound by the rate of random 128-B line fills (each account touch misses
    // L2), not by occupancy: more resident warps only lengthen the memory
    // queues and raise the abort rate (measured 0.300 / 0.312 / 0.331 ms per
    // 2^20-tx batch at 1 / 2 / 4 CTAs per SM).
    if (query_tx_occupancy(&b) != 0 || b < 1) return bail(fail(d, cudaErrorInvalidConfiguration, "batch kernel occupancy"));
    d->geom.max_blocks_tx = 1;
    d->geom.max_blocks_val = (query_val_occupancy(&b) == 0 && b > 0) ? b : 4;
    CK(d, cudaDeviceSynchronize());
    *out = d;
    return HETM_OK;
}

int hetm_dev_close(hetm_dev* d) {
    if (!d) return HETM_ERR_INVALID_ARG;
    cudaSetDevice(d->device);
    for (cudaStream_t s : {d->s_exec, d->s_copy, d->s_val, d->s_merge, d->s_d2h, d->s_zc, d->s_in, d->s_out, d->s_win})
        if (s) cudaStreamSynchronize(s);
    if (d->prep.active) {  // never merged: leave the host replica as it was
        std::lock_guard<std::mutex> g(d->mu);
        cancel_prepare(d);
    }
    d->pool.reset();
    for (int b = 0; b < 2; ++b) {
        if (d->h_delta[b].loc) cudaFreeHost(d->h_delta[b].loc);
        if (d->h_delta[b].val) cudaFreeHost(d->h_delta[b].val);
        for (cudaEvent_t e : d->piece_ev[b]) cudaEventDestroy(e);
    }
    for (cudaEvent_t e : d->in_ev) cudaEventDestroy(e);
    for (cudaEvent_t e : d->dl_ev) cudaEventDestroy(e);
    if (d->sched_graph.exec) cudaGraphExecDestroy(d->sched_graph.exec);
    if (d->sched_graph.graph) cudaGraphDestroy(d->sched_graph.graph);
    if (d->sched_graph.cap) cudaStreamDestroy(d->sched_graph.cap);
    if (d->s_est) {
        cudaStreamSynchronize(d->s_est);
        cudaStreamDestroy(d->s_est);
        cudaEventDestroy(d->ev_est);
        cudaFreeHost(d->h_hot);
    }
    for (cudaEvent_t e : d->kp_ev) cudaEventDestroy(e);
    for (void* p : {(void*)d->d_recv, (void*)d->d_recv_counts, (void*)d->d_peer_ptrs, (void*)d->d_peer_totals, (void*)d->d_res, (void*)d->d_wlog, (void*)d->d_delta[0].loc, (void*)d->d_delta[0].val, (void*)d->d_delta[1].loc, (void*)d->d_delta[1].val, (void*)d->ds.claim, (void*)d->ds.uniq, (void*)d->ds.uniq_val, (void*)d->ds.n_uniq, (void*)d->d_cells, (void*)d->d_shadow, (void*)d->d_stage, (void*)d->d_rs, (void*)d->d_ws,
                    (void*)d->d_chunk, (void*)d->d_ctr, (void*)d->d_pop, (void*)d->d_restore, (void*)d->d_arena, d->d_in,
                    (void*)d->d_tk, d->d_route, d->d_flush, (void*)d->d_trace, (void*)d->d_rs_zero, d->d_sched, (void*)d->d_est_in, (void*)d->d_stripes})
        if (p) cudaFree(p);
    if (d->h_ctr) cudaFreeHost(d->h_ctr);
    if (d->h_nrec) cudaFreeHost(d->h_nrec);
    if (d->ev_nrec) cudaEventDestroy(d->ev_nrec);
    if (d->ev_pick) cudaEventDestroy(d->ev_pick);
    if (d->h_first) cudaFreeHost(d->h_first);
    for (auto& v : d->tpairs)
        for (auto& pr : v) {
            cudaEventDestroy(pr.first);
            cudaEventDestroy(pr.second);
        }
    for (cudaEvent_t e : d->tpool) cudaEventDestroy(e);
    for (cudaStream_t s : {d->s_exec, d->s_copy, d->s_val, d->s_merge, d->s_d2h, d->s_zc, d->s_in, d->s_out, d->s_win})
        if (s) cudaStreamDestroy(s);
    for (cudaEvent_t e : {d->ev_exec, d->ev_copy, d->ev_val, d->ev_round, d->ev_shadow, d->ev_d2h, d->ev_t0, d->ev_t1,
                          d->ev_copy_zc, d->ev_stage, d->ev_ext, d->ev_win_fork, d->ev_win})
        if (e) cudaEventDestroy(e);
    delete d;
    return HETM_OK;
}

int hetm_dev_info_get(hetm_dev* d, hetm_dev_info* o) {
    if (!d || !o) return HETM_ERR_INVALID_ARG;
    std::memset(o, 0, sizeof(*o));
    o->size_words = d->W;
    o->shard_base = d->base;
    o->rs_gran_bytes = d->cfg.rs_gran_bytes;
    o->chunk_bytes = d->cfg.chunk_bytes;
    o->cell_bytes = sizeof(Cell);
    o->rs_bits = d->rs_bits;
    o->rs_words = d->rs_words;
    o->chunk_bits = d->chunk_bits;
    o->chunk_words = d->chunk_words;
    o->log_capacity = d->arena_cap;
    o->device_bytes = d->bytes_alloc;
    o->device = d->device;
    o->sm_count = d->geom.sm_count;
    o->l2_bytes = d->l2_bytes;
    int rc = sync_all(d);
    if (rc) return rc;
    if ((rc = read_counters(d))) return rc;
    o->ticket_next = d->h_ctr->ticket;
    return HETM_OK;
}

const char* hetm_dev_last_error(hetm_dev* d) { return d ? d->last_err.c_str() : "null handle"; }

// ------------------------------------------------------------ raw region ops
int hetm_dev_raw_write(hetm_dev* d, int replica, uint64_t addr, uint64_t value) {
    return hetm_dev_upload(d, replica, addr, &value, 1);
}

int hetm_dev_raw_read(hetm_dev* d, int replica, uint64_t addr, uint64_t* value) {
    if (!value) return HETM_ERR_INVALID_ARG;
    return hetm_dev_download(d, replica, addr, value, 1);
}

static int check_replica(hetm_dev* d, int replica) {
    if (replica == HETM_REPLICA_DEV) return HETM_OK;
    if (replica == HETM_REPLICA_DEV_SHADOW) return d->d_shadow ? HETM_OK : HETM_ERR_CONFIG;
    return HETM_ERR_INVALID_ARG;  // host-owned replicas are not addressable here
}

int hetm_dev_upload(hetm_dev* d, int replica, uint64_t addr, const uint64_t* src, uint64_t n) {
    if (!d || (!src && n)) return HETM_ERR_INVALID_ARG;
    int rc = check_replica(d, replica);
    if (rc) return rc;
    if ((rc = check_range(d, addr, n))) return rc;
    if ((rc = sync_all(d))) return rc;  // raw ops require quiescence
    const uint64_t lo = addr - d->base;
    if (replica == HETM_REPLICA_DEV_SHADOW) {
        CK(d, cudaMemcpy(d->d_shadow + lo, src, n * 8, cudaMemcpyHostToDevice));
    } else {
        if ((rc = ensure_stage(d, n))) return rc;
        CK(d, cudaMemcpy(d->d_stage, src, n * 8, cudaMemcpyHostToDevice));
        cudaError_t e = launch_scatter_range(d->d_cells, d->d_stage, lo, n, d->geom, 0);
        if (e == cudaSuccess) e = cudaDeviceSynchronize();
        if (e != cudaSuccess) return fail(d, e, "scatter_range");
    }
    d->shadow_synced = false;
    d->record(HETM_H2D, HETM_TAG_RAW, n * 8);
    return HETM_OK;
}

int hetm_dev_download(hetm_dev* d, int replica, uint64_t addr, uint64_t* dst, uint64_t n) {
    if (!d || (!dst && n)) return HETM_ERR_INVALID_ARG;
    int rc = check_replica(d, replica);
    if (rc) return rc;
    if ((rc = check_range(d, addr, n))) return rc;
    if ((rc = sync_all(d))) return rc;
    const uint64_t lo = addr - d->base;
    if (replica == HETM_REPLICA_DEV_SHADOW) {
        CK(d, cudaMemcpy(dst, d->d_shadow + lo, n * 8, cudaMemcpyDeviceToHost));
    } else {
        if ((rc = ensure_stage(d, n))) return rc;
        cudaError_t e = launch_gather_range(d->d_stage, d->d_cells, lo, n, d->geom, 0);
        if (e == cudaSuccess) e = cudaDeviceSynchronize();
        if (e != cudaSuccess) return fail(d, e, "gather_range");
        CK(d, cudaMemcpy(dst, d->d_stage, n * 8, cudaMemcpyDeviceToHost));
    }
    d->record(HETM_D2H, HETM_TAG_RAW, n * 8);
    return HETM_OK;
}

// ----------------------------------------------------------- batch execution
int hetm_dev_register_kernel(hetm_dev* d, int kernel_id) {
    if (!d) return HETM_ERR_INVALID_ARG;
    if (record_bytes(kernel_id) == 0) return HETM_ERR_NO_IMPLEMENTATION;
    d->kernels.insert(kernel_id);
    return HETM_OK;
}

int hetm_dev_execute_batch(hetm_dev* d, int kernel_id, const void* inputs, uint64_t rec_bytes, uint64_t n_tx,
                           uint64_t* tickets_out, hetm_batch_stats* stats) {
    return hetm_dev_execute_batch_ex(d, kernel_id, inputs, rec_bytes, n_tx, tickets_out, nullptr, 0, stats);
}

// Pieces of a host-input batch: one per 2^17 transactions, at most 8
// (HETM_EXEC_PIECES overrides, for experiments; 1 = unpipelined).
static uint64_t exec_pieces(uint64_t n_tx) {
    static const long want = [] {
        const char* e = std::getenv("HETM_EXEC_PIECES");
        return e ? std::atol(e) : 0L;
    }();
    uint64_t p = want > 0 ? (uint64_t)want : std::min<uint64_t>(8, n_tx >> 17);
    return std::max<uint64_t>(1, std::min<uint64_t>(p, std::max<uint64_t>(n_tx, 1)));
}

int hetm_dev_execute_batch_ex(hetm_dev* d, int kernel_id, const void* inputs, uint64_t rec_bytes, uint64_t n_tx,
                              uint64_t* tickets_out, void* results_out, uint64_t res_bytes,
                              hetm_batch_stats* stats) {
    NvtxRange nvtx_range("hetm.executeBatch");
    if (!d || (!inputs && n_tx)) return HETM_ERR_INVALID_ARG;
    if (!d->kernels.count(kernel_id)) return HETM_ERR_KERNEL_NOT_REGISTERED;
    if (rec_bytes != record_bytes(kernel_id)) return HETM_ERR_INVALID_SIZE;
    if (n_tx >= (1ull << 30)) return HETM_ERR_INVALID_SIZE;  // priorities are 30-bit
    if (results_out && (kernel_id != HETM_KERNEL_CACHE || res_bytes != sizeof(hetm_cache_result)))
        return HETM_ERR_INVALID_SIZE;
    int rc;
    if (results_out && n_tx > d->res_cap) {
        if (d->d_res) { CK(d, cudaStreamSynchronize(d->s_exec)); cudaFree(d->d_res); d->bytes_alloc -= d->res_cap * sizeof(hetm_cache_result); }
        d->res_cap = std::max<uint64_t>(n_tx, 1 << 16);
        if ((rc = dev_alloc(d, (void**)&d->d_res, d->res_cap * sizeof(hetm_cache_result)))) return rc;
    }
    if (n_tx * rec_bytes > d->in_cap) {
        if (d->d_in) { CK(d, cudaStreamSynchronize(d->s_exec)); cudaFree(d->d_in); d->bytes_alloc -= d->in_cap; }
        d->in_cap = std::max<uint64_t>(n_tx * rec_bytes, 1 << 20);
        if ((rc = dev_alloc(d, &d->d_in, d->in_cap))) return rc;
    }
    if (n_tx > d->tk_cap) {
        if (d->d_tk) { CK(d, cudaStreamSynchronize(d->s_exec)); cudaFree(d->d_tk); d->bytes_alloc -= d->tk_cap * 8; }
        d->tk_cap = std::max<uint64_t>(n_tx, 1 << 16);
        if ((rc = dev_alloc(d, (void**)&d->d_tk, d->tk_cap * 8))) return rc;
    }
    cudaStream_t s = d->s_exec;
    // first ticket of the batch, read after the batch's final sync (no extra host sync here)
    CK(d, cudaMemcpyAsync(d->h_first, &d->d_ctr->ticket, 8, cudaMemcpyDeviceToHost, s));
    CK(d, cudaMemsetAsync(&d->d_ctr->oob, 0, sizeof(unsigned), s));
    // Pipelined pieces: the H2D of piece k+1 (s_in) overlaps the kernel on
    // piece k (s_exec), whose tickets/results return on s_out while later
    // pieces run.  The pieces run back to back on s_exec, so the batch is
    // still one serializable execution (and input order in deterministic mode).
    const uint64_t P = exec_pieces(n_tx);
    while (d->in_ev.size() < P) {
        cudaEvent_t e = nullptr;
        CK(d, cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        d->in_ev.push_back(e);
    }
    while (d->kp_ev.size() < 2 * P) {
        cudaEvent_t e = nullptr;
        CK(d, cudaEventCreate(&e));
        d->kp_ev.push_back(e);
    }
    unsigned long long* trace = nullptr;  // armed checker trace (hetm_dev_trace_next_batch)
    if (d->trace_out && n_tx) {
        if (n_tx > d->trace_cap) {
            if (d->d_trace) { cudaFree(d->d_trace); d->bytes_alloc -= d->trace_cap * kTraceWords * 8; d->d_trace = nullptr; }
            if ((rc = dev_alloc(d, (void**)&d->d_trace, n_tx * kTraceWords * 8))) return rc;
            d->trace_cap = n_tx;
        }
        CK(d, cudaMemsetAsync(d->d_trace, 0xff, n_tx * kTraceWords * 8, s));  // ~0: did not commit
        trace = d->d_trace;
    }
    const char* in_h = static_cast<const char*>(inputs);
    char* in_d = static_cast<char*>(d->d_in);
    // every piece's H2D is queued first: the copies do not depend on the
    // schedule, so AUTO's host-side sample below runs while they stream (d_in
    // is free: the previous batch of this handle ended with a stream sync)
    for (uint64_t k = 0; k < P; ++k) {
        const uint64_t lo = n_tx * k / P, m = n_tx * (k + 1) / P - lo;
        if (!m) continue;
        CK(d, cudaMemcpyAsync(in_d + lo * rec_bytes, in_h + lo * rec_bytes, m * rec_bytes, cudaMemcpyHostToDevice,
                              d->s_in));
        CK(d, cudaEventRecord(d->in_ev[k], d->s_in));
    }
    d->dptr_feedback_n = 0;  // the counters now hold this batch's (judged below, synchronously)
    // AUTO for host-buffer bank batches: the CPU sample, or the retry feedback of
    // an earlier optimistic batch (judged at the end of this call: the pieces'
    // counters are read back anyway; zipf 0.5 in 8 pieces: SCAN 0.65 vs
    // optimistic 0.76 ms median, profiles/r02z_auto_feedback.txt)
    const bool auto_bank = kernel_id == HETM_KERNEL_BANK && d->schedule == HETM_SCHED_AUTO && n_tx;
    bool hot = false;
    if (auto_bank) {
        const bool feedback = d->auto_scan_left > 0;
        if (feedback) --d->auto_scan_left;
        hot = feedback || bank_batch_hot(static_cast<const hetm_bank_tx*>(inputs), n_tx);
    }
    // Kernel launches over the pieces: one per piece for the optimistic
    // kernels; the SCAN schedules pay fixed costs per launch (sort passes,
    // graph), so their pieces are grouped into two launches — the second half's
    // H2D still streams under the first half's kernels (zipf-0.5 bank batch:
    // 8 launches ~0.65 ms of kernel time, one ~0.31; profiles/r02al_*)
    const bool serial = (d->cfg.flags & HETM_CFG_DETERMINISTIC) != 0;
    const bool scan_path =
        (kernel_id == HETM_KERNEL_BANK && (serial || d->schedule == HETM_SCHED_SCAN || (auto_bank && hot))) ||
        (kernel_id == HETM_KERNEL_CACHE &&
         (serial || d->schedule == HETM_SCHED_SCAN || (d->schedule == HETM_SCHED_AUTO && n_tx / P >= kCacheScanMin)));
    const uint64_t G = scan_path ? std::min<uint64_t>(P, 2) : P;
    for (uint64_t k = 0; k < G; ++k) {
        const uint64_t p0 = P * k / G, p1 = P * (k + 1) / G;  // pieces [p0, p1) of this launch
        const uint64_t lo = n_tx * p0 / P, m = n_tx * p1 / P - lo;
        if (m) CK(d, cudaStreamWaitEvent(s, d->in_ev[p1 - 1], 0));  // s_in lands the pieces in order
        CK(d, cudaEventRecord(d->kp_ev[2 * k], s));
        if ((rc = enqueue_batch(d, kernel_id, in_d + lo * rec_bytes, m, d->d_tk + lo,
                                results_out ? d->d_res + lo : nullptr, s, k == 0,
                                trace ? trace + lo * kTraceWords : nullptr, hot)))
            return rc;
        CK(d, cudaEventRecord(d->kp_ev[2 * k + 1], s));
        if (m && (tickets_out || results_out)) {
            CK(d, cudaStreamWaitEvent(d->s_out, d->kp_ev[2 * k + 1], 0));
            if (tickets_out)
                CK(d, cudaMemcpyAsync(tickets_out + lo, d->d_tk + lo, m * 8, cudaMemcpyDeviceToHost, d->s_out));
            if (results_out)
                CK(d, cudaMemcpyAsync(static_cast<char*>(results_out) + lo * res_bytes, d->d_res + lo, m * res_bytes,
                                      cudaMemcpyDeviceToHost, d->s_out));
        }
    }
    if (n_tx) d->record(HETM_H2D, HETM_TAG_INPUT, n_tx * rec_bytes);
    if (tickets_out && n_tx) d->record(HETM_D2H, HETM_TAG_OUTPUT, n_tx * 8);
    if (results_out && n_tx) d->record(HETM_D2H, HETM_TAG_OUTPUT, n_tx * res_bytes);
    if (trace) {
        CK(d, cudaMemcpyAsync(d->trace_out, trace, n_tx * kTraceWords * 8, cudaMemcpyDeviceToHost, s));
        d->trace_out = nullptr;
    }
    CK(d, cudaMemcpyAsync(d->h_ctr, d->d_ctr, sizeof(DevCounters), cudaMemcpyDeviceToHost, s));
    CK(d, cudaStreamSynchronize(s));
    CK(d, cudaStreamSynchronize(d->s_out));
    float ms = 0.f;  // kernel time only: the sum over the launches
    for (uint64_t k = 0; k < G; ++k) {
        float mk = 0.f;
        cudaEventElapsedTime(&mk, d->kp_ev[2 * k], d->kp_ev[2 * k + 1]);
        ms += mk;
    }
    const uint64_t first = *d->h_first;
    hetm_batch_stats st{};
    st.n_tx = n_tx;
    st.committed = d->h_ctr->committed;
    st.aborts = d->h_ctr->aborts;
    st.retried = d->h_ctr->retried;
    st.livelocked = d->h_ctr->livelocked;
    st.ticket_first = first;
    st.ticket_end = d->h_ctr->ticket;
    st.kernel_ms = ms;
    d->last_batch = st;
    if (stats) *stats = st;
    if (auto_bank && !hot && !trace && st.retried * kAutoRetryRatio > n_tx) d->auto_scan_left = kAutoScanRun;
    if (d->h_ctr->oob) return HETM_ERR_OUT_OF_BOUNDS;
    if (st.livelocked) return HETM_ERR_LIVELOCK;
    return HETM_OK;
}

int hetm_dev_bitmap_words(hetm_dev* d, int which, uint64_t* n) {
    if (!d || !n) return HETM_ERR_INVALID_ARG;
    if (which == HETM_BMP_RS || which == HETM_BMP_WS) *n = d->rs_words;
    else if (which == HETM_BMP_CHUNK) *n = d->chunk_words;
    else return HETM_ERR_INVALID_ARG;
    return HETM_OK;
}

static unsigned long long* bitmap_ptr(hetm_dev* d, int which) {
    return which == HETM_BMP_RS ? d->d_rs : which == HETM_BMP_WS ? d->d_ws : which == HETM_BMP_CHUNK ? d->d_chunk : nullptr;
}

int hetm_dev_bitmap_stats(hetm_dev* d, uint64_t* rs, uint64_t* ws, uint64_t* chunks) {
    if (!d) return HETM_ERR_INVALID_ARG;
    int rc = sync_all(d);
    if (rc) return rc;
    CK(d, cudaMemset(d->d_pop, 0, 3 * 8));
    cudaError_t e;
    if ((e = launch_popcount(d->d_rs, d->rs_words, d->d_pop + 0, 0)) != cudaSuccess) return fail(d, e, "popcount");
    if ((e = launch_popcount(d->d_ws, d->rs_words, d->d_pop + 1, 0)) != cudaSuccess) return fail(d, e, "popcount");
    if ((e = launch_popcount(d->d_chunk, d->chunk_words, d->d_pop + 2, 0)) != cudaSuccess) return fail(d, e, "popcount");
    unsigned long long h[3];
    CK(d, cudaMemcpy(h, d->d_pop, 24, cudaMemcpyDeviceToHost));
    if (rs) *rs = h[0];
    if (ws) *ws = h[1];
    if (chunks) *chunks = h[2];
    return HETM_OK;
}

int hetm_dev_snapshot_bitmap(hetm_dev* d, int which, uint64_t* out, uint64_t n_words) {
    if (!d || !out) return HETM_ERR_INVALID_ARG;
    unsigned long long* p = bitmap_ptr(d, which);
    if (!p) return HETM_ERR_INVALID_ARG;
    uint64_t want = which == HETM_BMP_CHUNK ? d->chunk_words : d->rs_words;
    if (n_words != want) return HETM_ERR_INVALID_SIZE;
    int rc = sync_all(d);
    if (rc) return rc;
    CK(d, cudaMemcpy(out, p, n_words * 8, cudaMemcpyDeviceToHost));
    return HETM_OK;
}

int hetm_dev_bitmap_dptr(hetm_dev* d, int which, void** dptr, uint64_t* n_words) {
    if (!d || !dptr) return HETM_ERR_INVALID_ARG;
    unsigned long long* p = bitmap_ptr(d, which);
    if (!p) return HETM_ERR_INVALID_ARG;
    *dptr = p;
    if (n_words) *n_words = which == HETM_BMP_CHUNK ? d->chunk_words : d->rs_words;
    return HETM_OK;
}

int hetm_dev_bitmap_or_peers(hetm_dev* d, int which, const void* const* peer_words, uint32_t n_peers,
                             uint64_t word_lo, uint64_t word_hi, void* stream) {
    if (!d || (n_peers && !peer_words)) return HETM_ERR_INVALID_ARG;
    unsigned long long* p = bitmap_ptr(d, which);
    if (!p) return HETM_ERR_INVALID_ARG;
    const uint64_t n = which == HETM_BMP_CHUNK ? d->chunk_words : d->rs_words;
    if (word_hi == 0) word_hi = n;  // 0: the whole bitmap
    if (word_lo > word_hi || word_hi > n) return HETM_ERR_INVALID_SIZE;
    for (uint32_t k = 0; k < n_peers; ++k)
        if (!peer_words[k]) return HETM_ERR_INVALID_ARG;
    cudaStream_t s = stream ? static_cast<cudaStream_t>(stream) : d->s_val;
    CK(d, cudaStreamWaitEvent(s, d->ev_exec, 0));  // the local batches' bits are final
    cudaError_t e = launch_or_peers(p, reinterpret_cast<const unsigned long long* const*>(peer_words), n_peers,
                                    word_lo, word_hi, d->geom, s);
    if (e != cudaSuccess) return fail(d, e, "bitmap_or_peers");
    return join_val(d, s);
}

int hetm_dev_or_bitmap(hetm_dev* d, int which, const uint64_t* words, uint64_t n_words) {
    if (!d || (!words && n_words)) return HETM_ERR_INVALID_ARG;
    unsigned long long* p = bitmap_ptr(d, which);
    if (!p) return HETM_ERR_INVALID_ARG;
    uint64_t want = which == HETM_BMP_CHUNK ? d->chunk_words : d->rs_words;
    if (n_words != want) return HETM_ERR_INVALID_SIZE;
    int rc = sync_all(d);
    if (rc) return rc;
    void* tmp = nullptr;
    CK(d, cudaMalloc(&tmp, n_words * 8 + 8));
    cudaError_t e = cudaMemcpy(tmp, words, n_words * 8, cudaMemcpyHostToDevice);
    if (e == cudaSuccess) e = launch_or_words(p, static_cast<unsigned long long*>(tmp), n_words, 0);
    if (e == cudaSuccess) e = cudaDeviceSynchronize();
    cudaFree(tmp);
    if (e != cudaSuccess) return fail(d, e, "or_bitmap");
    return HETM_OK;
}

// --------------------------------------------------- log streaming / validation
int hetm_dev_open_intake(hetm_dev* d) {
    if (!d) return HETM_ERR_INVALID_ARG;
    std::lock_guard<std::mutex> g(d->mu);
    d->intake_open = true;
    return HETM_OK;
}

int hetm_dev_close_intake(hetm_dev* d) {
    if (!d) return HETM_ERR_INVALID_ARG;
    std::lock_guard<std::mutex> g(d->mu);
    d->intake_open = false;
    return HETM_OK;
}

// Validate-only launch over the pending early chunks [ev_lo, arena_n).
int flush_early_validation(hetm_dev* d) {
    if (d->ev_lo >= d->arena_n) {
        d->ev_pending = 0;
        return HETM_OK;
    }
    cudaError_t e = timed_validate(d, d->d_arena + d->ev_lo, d->arena_n - d->ev_lo, 0, d->s_val);
    if (e != cudaSuccess) return fail(d, e, "validate launch");
    CK(d, cudaMemcpyAsync(&d->h_ctr->conflict, &d->d_ctr->conflict, sizeof(unsigned), cudaMemcpyDeviceToHost,
                          d->s_val));
    d->ev_lo = d->arena_n;
    d->ev_pending = 0;
    return HETM_OK;
}

int hetm_dev_stream_chunk(hetm_dev* d, const hetm_log_entry* entries, uint64_t n, int src_thread, uint64_t seq,
                          int mode) {
    return hetm_dev_stream_chunk_ex(d, entries, n, src_thread, seq, mode, nullptr);
}

int hetm_dev_stream_chunk_ex(hetm_dev* d, const hetm_log_entry* entries, uint64_t n, int src_thread, uint64_t seq,
                             int mode, hetm_delivery* out) {
    NvtxRange nvtx_range("hetm.streamChunk");
    if (!d || (!entries && n) || src_thread < 0) return HETM_ERR_INVALID_ARG;
    if (mode != HETM_APPLY && mode != HETM_VALIDATE_ONLY) return HETM_ERR_INVALID_ARG;
    // One device-wide order for every chunk (the d->mu section): one source
    // thread's chunks are copied, validated and applied in the order its calls
    // return, which is the per-source FIFO of SPEC.md:300 (bus.hpp:80 streams
    // chunks of one thread's log in log order); different sources interleave in
    // arrival order ("validated in arbitrary order", §4.3).
    std::lock_guard<std::mutex> g(d->mu);
    if (!d->intake_open) return HETM_ERR_ROUND_CLOSED;
    d->record(HETM_H2D, HETM_TAG_LOG, n * sizeof(hetm_log_entry));
    // delivery handle: completion of this chunk's H2D copy (the host buffer is
    // the caller's again once it fires)
    if (d->dl_ev.empty()) {
        d->dl_ev.resize(kDeliveryRing, nullptr);
        for (auto& e : d->dl_ev) CK(d, cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    }
    const uint64_t h = d->dl_next++;
    cudaEvent_t ev = d->dl_ev[h % kDeliveryRing];
    if (h >= kDeliveryRing && d->dl_floor <= h - kDeliveryRing) {  // the slot's previous chunk: long delivered
        CK(d, cudaEventSynchronize(ev));
        d->dl_floor = h - kDeliveryRing + 1;
    }
    hetm_source_stats& src = d->sources[src_thread];
    src.chunks += 1;
    src.entries += n;
    src.last_seq = seq;
    src.last_handle = h;
    if (out) {
        out->seq = seq;
        out->n_entries = n;
        out->bytes = n * sizeof(hetm_log_entry);
        out->handle = h;
        out->src_thread = src_thread;
        out->mode = mode;
    }
    int rc;
    if (n == 0) {  // empty chunk: delivered at once (latency only)
        CK(d, cudaEventRecord(ev, d->s_copy));
        return HETM_OK;
    }
    if ((rc = ensure_arena(d, d->arena_n + n))) return rc;
    hetm_log_entry* dst = d->d_arena + d->arena_n;
    CK(d, cudaStreamWaitEvent(d->s_copy, d->ev_round, 0));
    CK(d, cudaMemcpyAsync(dst, entries, n * sizeof(hetm_log_entry), cudaMemcpyHostToDevice, d->s_copy));
    CK(d, cudaEventRecord(ev, d->s_copy));
    CK(d, cudaEventRecord(d->ev_copy, d->s_copy));
    CK(d, cudaStreamWaitEvent(d->s_val, d->ev_copy, 0));
    CK(d, cudaStreamWaitEvent(d->s_val, d->ev_round, 0));
    const bool apply = mode == HETM_APPLY;
    if (apply) {
        // pending early chunks are validated first (in arrival order)
        if ((rc = flush_early_validation(d))) return rc;
        if ((rc = ensure_restore(d, n))) return rc;
        CK(d, cudaStreamWaitEvent(d->s_val, d->ev_exec, 0));  // apply only after execution
        cudaError_t e = timed_validate(d, dst, n, 1, d->s_val);
        if (e != cudaSuccess) return fail(d, e, "validate launch");
        CK(d, cudaMemcpyAsync(&d->h_ctr->conflict, &d->d_ctr->conflict, sizeof(unsigned), cudaMemcpyDeviceToHost,
                              d->s_val));
        d->round_applied = true;
        d->arena_n += n;
        d->ev_lo = d->arena_n;
    } else {
        if (d->deferred.empty() || d->deferred.back().second != d->arena_n)
            d->deferred.emplace_back(d->arena_n, d->arena_n + n);
        else
            d->deferred.back().second += n;  // contiguous early chunks: one range
        d->deferred_final = false;
        d->arena_n += n;
        // early validation every ev_period chunks
        if (++d->ev_pending >= d->ev_period)
            if ((rc = flush_early_validation(d))) return rc;
    }
    return HETM_OK;
}

int hetm_dev_delivery_done(hetm_dev* d, uint64_t handle, int* done) {
    if (!d || !done) return HETM_ERR_INVALID_ARG;
    std::lock_guard<std::mutex> g(d->mu);
    if (handle >= d->dl_next) return HETM_ERR_INVALID_ARG;
    if (handle < d->dl_floor) {
        *done = 1;
        return HETM_OK;
    }
    const cudaError_t e = cudaEventQuery(d->dl_ev[handle % kDeliveryRing]);
    if (e == cudaErrorNotReady) {
        *done = 0;
        return HETM_OK;
    }
    if (e != cudaSuccess) return fail(d, e, "delivery query");
    *done = 1;
    d->dl_floor = std::max(d->dl_floor, handle + 1);  // s_copy completes in order
    return HETM_OK;
}

int hetm_dev_delivery_wait(hetm_dev* d, uint64_t handle) {
    if (!d) return HETM_ERR_INVALID_ARG;
    cudaEvent_t ev = nullptr;
    {
        std::lock_guard<std::mutex> g(d->mu);
        if (handle >= d->dl_next) return HETM_ERR_INVALID_ARG;
        if (handle < d->dl_floor) return HETM_OK;
        ev = d->dl_ev[handle % kDeliveryRing];
    }
    CK(d, cudaEventSynchronize(ev));
    std::lock_guard<std::mutex> g(d->mu);
    d->dl_floor = std::max(d->dl_floor, handle + 1);
    return HETM_OK;
}

int hetm_dev_source_stats(hetm_dev* d, int src_thread, hetm_source_stats* out) {
    if (!d || !out || src_thread < 0) return HETM_ERR_INVALID_ARG;
    std::lock_guard<std::mutex> g(d->mu);
    auto it = d->sources.find(src_thread);
    *out = it == d->sources.end() ? hetm_source_stats{} : it->second;
    return HETM_OK;
}

int hetm_dev_set_validation_period(hetm_dev* d, uint32_t k) {
    if (!d || k == 0) return HETM_ERR_INVALID_ARG;
    std::lock_guard<std::mutex> g(d->mu);
    d->ev_period = k;
    return HETM_OK;
}

int hetm_dev_apply_log(hetm_dev* d) {
    if (!d) return HETM_ERR_INVALID_ARG;
    std::lock_guard<std::mutex> g(d->mu);
    return enqueue_deferred_apply(d);
}

int hetm_dev_poll_conflict(hetm_dev* d, int* conflict) {
    if (!d || !conflict) return HETM_ERR_INVALID_ARG;
    *conflict = (int)*(volatile unsigned*)&d->h_ctr->conflict;
    return HETM_OK;
}

int hetm_dev_round_verdict(hetm_dev* d, int* conflict) {
    NvtxRange nvtx_range("hetm.roundVerdict");
    if (!d || !conflict) return HETM_ERR_INVALID_ARG;
    std::lock_guard<std::mutex> g(d->mu);
    // Chunks validated only early (possibly before the batch finished setting
    // its RS bits) are re-validated once execution has ended.
    d->ev_lo = d->arena_n;  // the final validation below covers the pending early chunks
    d->ev_pending = 0;
    if (!d->deferred.empty() && !d->deferred_final) {
        CK(d, cudaStreamWaitEvent(d->s_val, d->ev_exec, 0));
        for (auto& r : d->deferred) {
            cudaError_t e = timed_validate(d, d->d_arena + r.first, r.second - r.first, 0, d->s_val);
            if (e != cudaSuccess) return fail(d, e, "validate(final)");
        }
        d->deferred_final = true;
    }
    CK(d, cudaStreamSynchronize(d->s_copy));
    CK(d, cudaStreamSynchronize(d->s_val));
    int rc = read_counters(d);
    if (rc) return rc;
    *conflict = d->h_ctr->conflict ? 1 : 0;
    if (d->h_ctr->oob) return HETM_ERR_OUT_OF_BOUNDS;
    if (d->h_ctr->nonmonotone) return HETM_ERR_NONMONOTONE_TS;
    return HETM_OK;
}

int hetm_dev_sync(hetm_dev* d) {
    if (!d) return HETM_ERR_INVALID_ARG;
    return sync_all(d);
}

// ------------------------------------------------------------------- merge
namespace {
constexpr uint64_t kDeltaPiece = 1ull << 17;  // delta records per D2H piece (2 MiB)
static_assert(kDeltaPiece % 8192 == 0, "host scatter blocks must not straddle pieces");

// mergeCommit, delta form: the round's write-set log becomes a compact
// {word, value} list (16 B per written word instead of 16 KiB per dirty
// chunk), refreshed into devShadow on the device, DMA'd in pieces, and
// scattered into host_replica by the worker pool as each piece lands.  The
// host replica ends identical to the chunk copy: the words outside the device
// write set inside a dirty chunk already hold the host's values (the round
// committed, so no host entry touched a device-read word).
// Grow the delta buffers to hold n_slots records (records <= slots), the
// pinned landing buffers with them, and the claim bitmap (W bits, kept zero
// between stages by the emit kernel).
int ensure_delta(hetm_dev* d, uint64_t n_slots) {
    if (!d->ds.claim) {
        const uint64_t words = (d->W + 63) / 64;
        if (int rc = dev_alloc(d, (void**)&d->ds.claim, words * 8)) return rc;
        CK(d, cudaMemset(d->ds.claim, 0, words * 8));
        // records, slots (pick pass), then the bucket counts/cursors: one allocation, one memset per stage
        constexpr size_t kCtrPad = 256, kBuckets = 2 * kDeltaBuckets * sizeof(uint32_t);
        if (int rc = dev_alloc(d, (void**)&d->ds.n_uniq, kCtrPad + kBuckets)) return rc;
        d->ds.bucket_cnt = reinterpret_cast<uint32_t*>(reinterpret_cast<char*>(d->ds.n_uniq) + kCtrPad);
        d->ds.counters_bytes = kCtrPad + kBuckets;
        if (cudaHostAlloc((void**)&d->h_nrec, 64, cudaHostAllocPortable) != cudaSuccess)
            return fail(d, cudaGetLastError(), "cudaHostAlloc(record count)");
        CK(d, cudaEventCreateWithFlags(&d->ev_nrec, cudaEventDisableTiming));
        CK(d, cudaEventCreateWithFlags(&d->ev_pick, cudaEventDisableTiming));
    }
    if (n_slots <= d->delta_cap) return HETM_OK;
    if (d->pool) d->pool->wait();  // nothing may still read the old buffers
    CK(d, cudaStreamSynchronize(d->s_merge));
    CK(d, cudaStreamSynchronize(d->s_d2h));
    for (int b = 0; b < 2; ++b) {
        if (d->d_delta[b].loc) { cudaFree(d->d_delta[b].loc); cudaFree(d->d_delta[b].val); d->bytes_alloc -= d->delta_cap * 12; }
        if (d->h_delta[b].loc) { cudaFreeHost(d->h_delta[b].loc); cudaFreeHost(d->h_delta[b].val); }
        d->d_delta[b] = DeltaBuf{nullptr, nullptr};
        d->h_delta[b] = DeltaBuf{nullptr, nullptr};
    }
    if (d->ds.uniq) { cudaFree(d->ds.uniq); d->bytes_alloc -= d->delta_cap * 4; d->ds.uniq = nullptr; }
    if (d->ds.uniq_val) { cudaFree(d->ds.uniq_val); d->bytes_alloc -= d->delta_cap * 8; d->ds.uniq_val = nullptr; }
    const uint64_t cap = std::max<uint64_t>(n_slots + n_slots / 4, 1ull << 21);  // pinning is slow: grow rarely
    for (int b = 0; b < 2; ++b) {
        if (int rc = dev_alloc(d, (void**)&d->d_delta[b].loc, cap * 4)) return rc;
        if (int rc = dev_alloc(d, (void**)&d->d_delta[b].val, cap * 8)) return rc;
        if (cudaHostAlloc((void**)&d->h_delta[b].loc, cap * 4, cudaHostAllocPortable) != cudaSuccess ||
            cudaHostAlloc((void**)&d->h_delta[b].val, cap * 8, cudaHostAllocPortable) != cudaSuccess)
            return fail(d, cudaGetLastError(), "cudaHostAlloc(delta)");
    }
    if (int rc = dev_alloc(d, (void**)&d->ds.uniq, cap * 4)) return rc;
    if (int rc = dev_alloc(d, (void**)&d->ds.uniq_val, cap * 8)) return rc;
    d->delta_cap = cap;
    return HETM_OK;
}

// Device half of the delta merge, on s_merge: the round's n_slots write-set
// log slots become one {word, value} record per written word in delta buffer
// `buf` (claim + emit kernels, no sort), devShadow refreshed with the same
// values when shadow != nullptr.  The record count lands in h_nrec (ev_nrec).
int stage_records(hetm_dev* d, uint64_t n_slots, uint64_t* shadow, int buf) {
    if (int rc = ensure_delta(d, n_slots)) return rc;
    const bool picked = d->round_versioned;
    cudaError_t e = picked ? launch_delta_pick(d->d_wlog, n_slots, d->W, d->d_cells, d->ds, d->geom, d->s_merge,
                                               d->d_ctr, false)
                           : launch_delta_claim(d->d_wlog, n_slots, d->W, d->ds, d->geom, d->s_merge);
    if (e != cudaSuccess) return fail(d, e, "delta_claim");
    CK(d, cudaMemcpyAsync(d->h_nrec, d->ds.n_uniq, 8, cudaMemcpyDeviceToHost, d->s_merge));
    CK(d, cudaEventRecord(d->ev_nrec, d->s_merge));
    e = launch_delta_emit(n_slots, d->W, d->ds, d->d_cells, d->d_delta[buf], shadow, d->geom, d->s_merge, picked);
    if (e != cudaSuccess) return fail(d, e, "delta_emit");
    CK(d, cudaEventRecord(d->ev_stage, d->s_merge));
    return HETM_OK;
}

// The other delta buffer (the one the worker pool is not scattering from) and
// the host worker pool, created on first use.
int next_delta_buffer(hetm_dev* d) {
    const int b = d->dbuf;
    d->dbuf ^= 1;
    if (!d->pool) {
        // this process's share of the usable cores (torchrun runs one process
        // per GPU: LOCAL_WORLD_SIZE), one core left to the controller thread
        // (it spin-waits on CUDA)
        static const unsigned want = [] {
            const char* e = std::getenv("HETM_MERGE_THREADS");
            return e ? (unsigned)std::atoi(e) : 0u;
        }();
        unsigned cores = std::thread::hardware_concurrency();
        cpu_set_t cs;
        if (sched_getaffinity(0, sizeof(cs), &cs) == 0) cores = (unsigned)CPU_COUNT(&cs);
        const char* lws = std::getenv("LOCAL_WORLD_SIZE");
        const unsigned procs = lws ? std::max(1, std::atoi(lws)) : 1u;
        const unsigned share = std::max(1u, (cores ? cores : 4u) / procs);
        const unsigned n = want ? want : std::min(32u, share > 1 ? share - 1 : 1u);
        d->pool.reset(new WorkerPool((int)std::max(1u, n)));
    }
    return b;
}

// Host half: DMA the staged records of `buf` in pieces (each with a completion
// event), after their count is known; the first n_zc records optionally go
// into the mapped host replica as zero-copy stores instead.
int ship_records(hetm_dev* d, int buf, uint64_t* zc_host, uint64_t* n_rec_out, uint64_t* k0_out,
                 uint64_t* pieces_out, uint64_t* bytes_d2h) {
    CK(d, cudaEventSynchronize(d->ev_nrec));  // the claim pass is done (~15 us after the batch)
    const uint64_t n_rec = *reinterpret_cast<volatile uint64_t*>(d->h_nrec);
    const DeltaBuf dd = d->d_delta[buf];
    const DeltaBuf hd = d->h_delta[buf];
    std::vector<cudaEvent_t>& pev = d->piece_ev[buf];
    CK(d, cudaStreamWaitEvent(d->s_d2h, d->ev_stage, 0));
    uint64_t n_zc = 0;
    if (zc_host) {
        // Split: the first n_zc records are stored into the host replica by the
        // GPU itself (zero-copy PCIe writes, s_zc) while the copy engine and the
        // host workers deliver the rest — two independent paths.
        static const double zc_frac = [] {
            const char* e = std::getenv("HETM_ZC_FRACTION");
            // 0 since the host scatter prefetches: the zero-copy stores then only
            // slow the next batch's input H2D (profiles/r01_e2e_timeline.txt)
            return e ? std::atof(e) : 0.0;
        }();
        cudaPointerAttributes pa{};
        if (zc_frac > 0 && cudaPointerGetAttributes(&pa, zc_host) == cudaSuccess && pa.type == cudaMemoryTypeHost &&
            pa.devicePointer) {
            n_zc = std::min<uint64_t>(n_rec, (uint64_t)(zc_frac * (double)n_rec)) / kDeltaPiece * kDeltaPiece;
            if (n_zc) {
                CK(d, cudaStreamWaitEvent(d->s_zc, d->ev_stage, 0));
                cudaError_t ez = launch_delta_zc_scatter(static_cast<uint64_t*>(pa.devicePointer), dd, n_zc,
                                                         d->geom, d->s_zc);
                if (ez != cudaSuccess) return fail(d, ez, "delta_zc_scatter");
                d->record(HETM_D2H, HETM_TAG_MERGE_DELTA, n_zc * 8);
            }
        } else {
            cudaGetLastError();
        }
    }
    const uint64_t pieces = (n_rec + kDeltaPiece - 1) / kDeltaPiece;
    while (pev.size() < pieces) {
        cudaEvent_t ev = nullptr;
        CK(d, cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
        pev.push_back(ev);
    }
    const uint64_t k0 = n_zc / kDeltaPiece;  // pieces already delivered by the zero-copy kernel
    for (uint64_t k = k0; k < pieces; ++k) {
        const uint64_t lo = k * kDeltaPiece, m = std::min(kDeltaPiece, n_rec - lo);
        CK(d, cudaMemcpyAsync(hd.loc + lo, dd.loc + lo, m * 4, cudaMemcpyDeviceToHost, d->s_d2h));
        CK(d, cudaMemcpyAsync(hd.val + lo, dd.val + lo, m * 8, cudaMemcpyDeviceToHost, d->s_d2h));
        CK(d, cudaEventRecord(pev[k], d->s_d2h));
    }
    d->record(HETM_D2H, HETM_TAG_MERGE_DELTA, (n_rec - n_zc) * 12);
    *bytes_d2h = n_zc * 8 + (n_rec - n_zc) * 12;
    if (n_zc) {  // the merge is complete when both paths are
        CK(d, cudaEventRecord(d->ev_copy_zc, d->s_zc));
        CK(d, cudaStreamWaitEvent(d->s_d2h, d->ev_copy_zc, 0));
    }
    CK(d, cudaEventRecord(d->ev_d2h, d->s_d2h));
    d->d2h_pending = true;
    *n_rec_out = n_rec;
    *k0_out = k0;
    *pieces_out = pieces;
    return HETM_OK;
}

// Host side of the delta: the worker pool writes the records into the host
// replica as each DMA piece lands.  PLAIN stores them; SWAP (speculative, before
// the round's verdict) stores them and keeps the replaced value in the record,
// so UNDO can put the replica back (records are unique per word).
enum ScatterMode { kScatterPlain, kScatterSwap, kScatterUndo };

void start_scatter(hetm_dev* d, int buf, uint64_t* host, uint64_t n_rec, uint64_t k0, uint64_t pieces,
                   ScatterMode mode) {
    const DeltaBuf src = d->h_delta[buf];
    const std::vector<cudaEvent_t> evs(d->piece_ev[buf].begin(), d->piece_ev[buf].begin() + pieces);
    const int dev = d->device;
    // Dynamic blocks in sorted order: a worker that the OS deschedules delays
    // only the block it holds, not a static 1/nw share of every piece.  Piece
    // arrival is polled by one worker at a time (cudaEventQuery under a
    // try-lock) and published through `landed`.
    struct ScatterState {
        std::atomic<uint64_t> cursor{0};  // next record to claim
        std::atomic<uint64_t> landed{0};  // pieces known to be in h_delta
        std::mutex waiter;                // one worker at a time polls the driver
    };
    auto st = std::make_shared<ScatterState>();
    st->cursor = k0 * kDeltaPiece;
    st->landed = mode == kScatterUndo ? pieces : k0;  // undo runs on records already in place
    d->pool->start([src, evs, host, n_rec, dev, st, mode](int, int) {
        cudaSetDevice(dev);
        constexpr uint64_t kBlock = 8192;   // records per claim (divides kDeltaPiece)
        constexpr uint64_t kPrefetch = 64;  // prefetch-for-write distance, see below
        for (;;) {
            const uint64_t a = st->cursor.fetch_add(kBlock, std::memory_order_relaxed);
            if (a >= n_rec) return;
            const uint64_t b = std::min(a + kBlock, n_rec), k = a / kDeltaPiece;
            while (st->landed.load(std::memory_order_acquire) <= k) {
                if (st->waiter.try_lock()) {  // the others spin on `landed`, not in the driver
                    // block on the next missing piece: a tight cudaEventQuery loop
                    // would contend with the controller thread's CUDA calls
                    uint64_t l = st->landed.load(std::memory_order_relaxed);
                    if (l <= k) {
                        cudaEventSynchronize(evs[l]);
                        ++l;
                        while (l <= k && cudaEventQuery(evs[l]) == cudaSuccess) ++l;
                    }
                    st->landed.store(l, std::memory_order_release);
                    st->waiter.unlock();
                }
                std::this_thread::yield();
            }
            // x86 drains stores in order, so without the prefetch the random RFO
            // misses serialise (3.3 vs 1.8 G words/s on the box's 16 cores,
            // profiles/r01_host_scatter_probe.txt)
            for (uint64_t i = a; i < b; ++i) {
                if (i + kPrefetch < b && src.loc[i + kPrefetch] != ~0u)
                    __builtin_prefetch(&host[src.loc[i + kPrefetch]], 1, 0);
                const uint32_t loc = src.loc[i];
                if (loc == ~0u) continue;
                if (mode == kScatterSwap) {
                    const uint64_t old = host[loc];
                    host[loc] = src.val[i];
                    src.val[i] = old;
                } else {
                    host[loc] = src.val[i];
                }
            }
        }
    });
}

// A prepared merge that will not be committed (a conflict, a new batch, a
// clear): wait for its host side and undo a speculative scatter.
void cancel_prepare(hetm_dev* d) {
    if (!d->prep.active) return;
    d->pool->wait();
    if (d->prep.speculative) {
        start_scatter(d, d->prep.buf, d->prep.host, d->prep.n_rec, d->prep.k0, d->prep.pieces, kScatterUndo);
        d->pool->wait();
    }
    d->prep = PreparedMerge{};
}

// Delta mergeCommit: the batch kernels logged the word index of every
// committed write into the slot of its commit ticket; the log is sorted and
// gathered into {word, value} records (devShadow refreshed with them), DMA'd
// in 2 MiB pieces and scattered into host_replica by the worker pool as each
// piece lands.  The host replica ends identical to the chunk copy: the words
// outside the device write set inside a dirty chunk already hold the host's
// values (the round committed, so no host entry touched a device-read word).
// After hetm_dev_merge_prepare the records are already staged (and, when it
// got the host replica, already in it): only the shadow is refreshed here.
int merge_commit_delta(hetm_dev* d, uint64_t* host, uint64_t n_slots, uint64_t* bytes_d2h, uint64_t* n_rec_out) {
    const bool prepared = d->prep.active && d->prep.round_tx == d->round_tx && d->prep.n_slots == n_slots;
    const bool staged = !prepared && d->staged.active && d->staged.round_tx == d->round_tx;
    if (!prepared && d->d2h_pending) CK(d, cudaStreamWaitEvent(d->s_merge, d->ev_d2h, 0));  // the previous delta
    // shadow: incremental when it held the round-start state, else a full copy
    uint64_t* shadow_inc = (d->d_shadow && d->shadow_synced) ? d->d_shadow : nullptr;
    if (d->d_shadow && !d->shadow_synced) {
        cudaError_t e = launch_dirty_chunks(d->d_shadow, d->d_cells, d->W, nullptr, d->chunk_bits, d->chunk_shift, true,
                                            d->geom, d->s_merge);
        if (e != cudaSuccess) return fail(d, e, "dirty_chunks(full shadow)");
        d->record(HETM_D2D, HETM_TAG_SHADOW, d->W * 8);
        d->shadow_synced = true;
    }
    if (prepared) {
        const PreparedMerge p = d->prep;
        d->prep = PreparedMerge{};
        if (shadow_inc) {
            cudaError_t e = launch_delta_to_shadow(shadow_inc, d->d_delta[p.buf], p.n_rec, d->geom, d->s_merge);
            if (e == cudaSuccess) e = patch_shadow(d);
            if (e != cudaSuccess) return fail(d, e, "shadow(prepared merge)");
            d->record(HETM_D2D, HETM_TAG_SHADOW, p.n_rec * 8);
        }
        CK(d, cudaEventRecord(d->ev_shadow, d->s_merge));
        if (!p.speculative || p.host != host) {
            if (p.speculative) {  // prepared for another replica: put that one back first
                d->pool->wait();
                start_scatter(d, p.buf, p.host, p.n_rec, p.k0, p.pieces, kScatterUndo);
                d->pool->wait();
                for (uint64_t k = 0; k < p.pieces; ++k) {  // the records hold old values now: restage
                    const uint64_t lo = k * kDeltaPiece, m = std::min(kDeltaPiece, p.n_rec - lo);
                    CK(d, cudaMemcpyAsync(d->h_delta[p.buf].val + lo, d->d_delta[p.buf].val + lo, m * 8,
                                          cudaMemcpyDeviceToHost, d->s_d2h));
                    CK(d, cudaEventRecord(d->piece_ev[p.buf][k], d->s_d2h));
                }
            }
            start_scatter(d, p.buf, host, p.n_rec, p.k0, p.pieces, kScatterPlain);
        }
        *bytes_d2h = p.n_rec * 12;
        *n_rec_out = p.n_rec;
        return HETM_OK;
    }
    cancel_prepare(d);
    int buf;
    if (staged) {  // hetm_dev_merge_stage did the device half (records + shadow) already
        buf = d->staged.buf;
        d->staged.active = false;
    } else {
        buf = next_delta_buffer(d);
        if (int rc = stage_records(d, n_slots, shadow_inc, buf)) return rc;
        if (shadow_inc) {
            cudaError_t e = patch_shadow(d);
            if (e != cudaSuccess) return fail(d, e, "winner_apply(shadow)");
        }
        CK(d, cudaEventRecord(d->ev_shadow, d->s_merge));
    }
    uint64_t n_rec = 0, k0 = 0, pieces = 0;
    if (int rc = ship_records(d, buf, host, &n_rec, &k0, &pieces, bytes_d2h)) return rc;
    if (shadow_inc && !staged) d->record(HETM_D2D, HETM_TAG_SHADOW, n_rec * 8);
    start_scatter(d, buf, host, n_rec, k0, pieces, kScatterPlain);
    *n_rec_out = n_rec;
    return HETM_OK;
}
}  // namespace

int hetm_dev_merge_commit(hetm_dev* d, uint64_t* host, hetm_merge_stats* st) {
    NvtxRange nvtx_range("hetm.mergeCommit");
    if (!d || !host) return HETM_ERR_INVALID_ARG;
    auto t0 = std::chrono::steady_clock::now();
    std::lock_guard<std::mutex> g(d->mu);
    d->intake_open = false;  // merge closes the log intake
    if (!d->deferred.empty()) return HETM_ERR_STATE;  // all chunks must be applied
    int rc = wait_round_work(d, d->s_merge);
    if (rc) return rc;
    CK(d, cudaStreamSynchronize(d->s_exec));
    CK(d, cudaStreamSynchronize(d->s_val));
    if ((rc = read_counters(d))) return rc;
    if (d->h_ctr->conflict) return HETM_ERR_STATE;  // pre: conflictFlag = false
    std::vector<std::pair<uint64_t, uint64_t>> ranges;
    uint64_t nd = 0;
    if ((rc = dirty_ranges(d, ranges, &nd))) return rc;
    uint64_t dirty_bytes = 0;
    for (auto& r : ranges) dirty_bytes += r.second * 8;
    // delta form when enabled, the write-set log is complete and it moves fewer bytes
    const uint64_t n_slots = 2 * (d->h_ctr->ticket - d->h_ctr->wlog_base);
    // (a merge prepared for this round has its records in flight or already in
    // the host replica: it completes as a delta whatever the byte counts)
    const bool prepared = d->prep.active && d->prep.round_tx == d->round_tx && d->prep.n_slots == n_slots;
    const bool delta = (d->cfg.flags & HETM_CFG_MERGE_DELTA) && d->d_wlog && !d->h_ctr->wlog_overflow &&
                       n_slots <= d->wlog_slots && (prepared || n_slots * 12 < dirty_bytes);
    if (delta) {
        uint64_t moved = 0, n_rec = 0;
        if ((rc = merge_commit_delta(d, host, n_slots, &moved, &n_rec))) return rc;
        if (st) {
            std::memset(st, 0, sizeof(*st));
            st->dirty_chunks = nd;
            st->transfers = (n_rec + kDeltaPiece - 1) / kDeltaPiece;
            st->bytes_d2h = moved;
            st->bytes_d2d = d->d_shadow ? n_rec * 8 : 0;
            st->ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
        }
        return HETM_OK;
    }
    cancel_prepare(d);             // a stale prepared delta (another round) is undone first
    if (d->pool) d->pool->wait();  // a previous delta merge may still be landing in host_replica
    const uint64_t* src = d->d_shadow;
    if (d->d_shadow) {
        if ((rc = refresh_shadow(d, true, dirty_bytes))) return rc;
    } else {  // no shadow: pack the dirty chunks into the staging buffer instead
        if ((rc = ensure_stage(d, d->W))) return rc;
        cudaError_t e = launch_dirty_chunks(d->d_stage, d->d_cells, d->W, d->d_chunk, d->chunk_bits, d->chunk_shift,
                                            true, d->geom, d->s_merge);
        if (e != cudaSuccess) return fail(d, e, "dirty_chunks(stage)");
        CK(d, cudaEventRecord(d->ev_shadow, d->s_merge));
        src = d->d_stage;
    }
    CK(d, cudaStreamWaitEvent(d->s_d2h, d->ev_shadow, 0));
    for (auto& r : ranges) {
        CK(d, cudaMemcpyAsync(host + r.first, src + r.first, r.second * 8, cudaMemcpyDeviceToHost, d->s_d2h));
        d->record(HETM_D2H, HETM_TAG_MERGE, r.second * 8);
    }
    CK(d, cudaEventRecord(d->ev_d2h, d->s_d2h));
    d->d2h_pending = true;
    if (!d->d_shadow) CK(d, cudaStreamSynchronize(d->s_d2h));  // no double buffer without a shadow
    if (st) {
        std::memset(st, 0, sizeof(*st));
        st->dirty_chunks = nd;
        st->transfers = ranges.size();
        st->bytes_d2h = dirty_bytes;
        st->bytes_d2d = d->d_shadow ? dirty_bytes : 0;
        st->ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    }
    return HETM_OK;
}

int hetm_dev_merge_prepare(hetm_dev* d, uint64_t* host) {
    NvtxRange nvtx_range("hetm.mergePrepare");
    if (!d) return HETM_ERR_INVALID_ARG;
    std::lock_guard<std::mutex> g(d->mu);
    cancel_prepare(d);
    if (!(d->cfg.flags & HETM_CFG_MERGE_DELTA) || !d->d_wlog) return HETM_OK;  // chunk merge: nothing to stage
    CK(d, cudaStreamSynchronize(d->s_exec));  // the execution phase is over
    int rc = read_counters(d);
    if (rc) return rc;
    const uint64_t n_slots = 2 * (d->h_ctr->ticket - d->h_ctr->wlog_base);
    if (d->h_ctr->wlog_overflow || n_slots == 0 || n_slots > d->wlog_slots) return HETM_OK;
    // staged into the other delta buffer while the pool may still scatter the
    // previous round's; starting this round's job below waits for that one, so
    // host transactions after this call see the previous merge landed
    CK(d, cudaStreamWaitEvent(d->s_merge, d->ev_exec, 0));
    if (d->d2h_pending) CK(d, cudaStreamWaitEvent(d->s_merge, d->ev_d2h, 0));  // the previous delta's DMA
    uint64_t k0 = 0, pieces = 0, moved = 0, n_rec = 0;
    const int buf = next_delta_buffer(d);
    d->staged.active = false;
    if ((rc = stage_records(d, n_slots, nullptr, buf))) return rc;
    if ((rc = ship_records(d, buf, nullptr, &n_rec, &k0, &pieces, &moved))) return rc;
    d->prep.active = true;
    d->prep.speculative = host != nullptr;
    d->prep.n_slots = n_slots;
    d->prep.n_rec = n_rec;
    d->prep.k0 = k0;
    d->prep.pieces = pieces;
    d->prep.round_tx = d->round_tx;
    d->prep.host = host;
    d->prep.buf = buf;
    if (host) start_scatter(d, buf, host, n_rec, k0, pieces, kScatterSwap);
    else if (d->pool) d->pool->wait();  // still: the previous merge has landed when this returns
    return HETM_OK;
}

int hetm_dev_merge_stage(hetm_dev* d) {
    NvtxRange nvtx_range("hetm.mergeStage");
    if (!d) return HETM_ERR_INVALID_ARG;
    std::lock_guard<std::mutex> g(d->mu);
    if (!(d->cfg.flags & HETM_CFG_MERGE_DELTA) || !d->d_wlog) return HETM_ERR_CONFIG;
    if (!d->deferred.empty()) return HETM_ERR_STATE;  // every chunk must be applied first
    cancel_prepare(d);
    d->intake_open = false;  // the merge has started
    d->merge_staged = true;
    int rc = wait_round_work(d, d->s_merge);  // the batches and the validation of the round
    if (rc) return rc;
    if (d->d2h_pending) CK(d, cudaStreamWaitEvent(d->s_merge, d->ev_d2h, 0));  // the previous delta's DMA
    uint64_t* shadow_inc = (d->d_shadow && d->shadow_synced) ? d->d_shadow : nullptr;
    if (d->d_shadow && !d->shadow_synced) {  // gated on the host at merge_commit instead (full copy)
        d->staged.active = false;
        return HETM_OK;
    }
    const int buf = next_delta_buffer(d);
    // the slot count and the verdict are read by the kernels themselves: on a
    // conflict (or a write-set log overflow) they stage nothing and leave
    // devShadow at the round start, so mergeAbortDevice stays exact
    if ((rc = ensure_delta(d, d->wlog_slots))) return rc;  // records <= slots in use <= capacity
    cudaEvent_t t0 = nullptr, t1 = nullptr;
    if (d->timing) {
        t0 = d->tev();
        t1 = d->tev();
        CK(d, cudaEventRecord(t0, d->s_merge));
    }
    // the winner patch touches only host-log words, the pick/emit only device-
    // written ones: in a committed round the two sets are disjoint (WS within RS,
    // no RS/host-write intersection), and both are verdict-gated on the device
    const bool win_side = shadow_inc && d->win_side;
    if (win_side) {
        CK(d, cudaEventRecord(d->ev_win_fork, d->s_merge));
        CK(d, cudaStreamWaitEvent(d->s_win, d->ev_win_fork, 0));
        cudaError_t ew = patch_shadow(d, d->d_ctr, d->s_win);
        if (ew != cudaSuccess) return fail(d, ew, "winner_apply(stage)");
        CK(d, cudaEventRecord(d->ev_win, d->s_win));
    }
    const bool picked = d->round_versioned;
    cudaError_t e = picked ? launch_delta_pick(d->d_wlog, d->wlog_slots, d->W, d->d_cells, d->ds, d->geom,
                                               d->s_merge, d->d_ctr, true)
                           : launch_delta_claim(d->d_wlog, d->wlog_slots, d->W, d->ds, d->geom, d->s_merge, d->d_ctr);
    if (e != cudaSuccess) return fail(d, e, "delta_claim(stage)");
    // the record count goes to the host on a side stream, so the copy does not
    // sit between the pick and the emit on s_merge
    CK(d, cudaEventRecord(d->ev_pick, d->s_merge));
    CK(d, cudaStreamWaitEvent(d->s_zc, d->ev_pick, 0));
    CK(d, cudaMemcpyAsync(d->h_nrec, d->ds.n_uniq, 8, cudaMemcpyDeviceToHost, d->s_zc));
    CK(d, cudaEventRecord(d->ev_nrec, d->s_zc));
    // (running the emit beside the next round's batch was measured slower: its
    // random shadow stores and the batch's random accesses share the DRAM)
    e = launch_delta_emit(d->wlog_slots, d->W, d->ds, d->d_cells, d->d_delta[buf], shadow_inc, d->geom, d->s_merge,
                          picked);
    if (e != cudaSuccess) return fail(d, e, "delta_emit(stage)");
    CK(d, cudaEventRecord(d->ev_stage, d->s_merge));
    if (win_side) CK(d, cudaStreamWaitEvent(d->s_merge, d->ev_win, 0));
    else if (shadow_inc && (e = patch_shadow(d, d->d_ctr)) != cudaSuccess) return fail(d, e, "winner_apply(stage)");
    if (d->timing) {
        CK(d, cudaEventRecord(t1, d->s_merge));
        d->tpairs[2].emplace_back(t0, t1);
    }
    CK(d, cudaEventRecord(d->ev_shadow, d->s_merge));
    d->staged.active = true;
    d->staged.round_tx = d->round_tx;
    d->staged.buf = buf;
    return HETM_OK;
}

int hetm_dev_merge_abort_device(hetm_dev* d, int optimized, const uint64_t* host, hetm_merge_stats* st) {
    NvtxRange nvtx_range("hetm.mergeAbortDevice");
    if (!d || (!host && !optimized)) return HETM_ERR_INVALID_ARG;
    auto t0 = std::chrono::steady_clock::now();
    std::lock_guard<std::mutex> g(d->mu);
    cancel_prepare(d);  // undo a speculative delta first: the device side of the round is void
    d->intake_open = false;
    int rc = enqueue_deferred_apply(d);  // FavorHost: the host log always lands on the device
    if (rc) return rc;
    if ((rc = wait_round_work(d, d->s_merge))) return rc;
    CK(d, cudaStreamSynchronize(d->s_exec));
    CK(d, cudaStreamSynchronize(d->s_val));
    std::vector<std::pair<uint64_t, uint64_t>> ranges;
    uint64_t nd = 0;
    if ((rc = dirty_ranges(d, ranges, &nd))) return rc;
    uint64_t dirty_bytes = 0;
    for (auto& r : ranges) dirty_bytes += r.second * 8;
    if (d->d2h_pending) CK(d, cudaStreamWaitEvent(d->s_merge, d->ev_d2h, 0));
    hetm_merge_stats s{};
    if (optimized && d->d_shadow && d->shadow_synced) {
        // Round-start shadow + the round's host log in ts order: the
        // device-dirty words are restored from devShadow (just the device write
        // set when the write-set log holds it, else whole dirty chunks), then the
        // freshest log entry of every logged word is stored into both devReplica
        // and devShadow.
        if ((rc = read_counters(d))) return rc;
        const uint64_t n_slots = 2 * (d->h_ctr->ticket - d->h_ctr->wlog_base);
        cudaError_t e;
        if (d->d_wlog && !d->h_ctr->wlog_overflow && n_slots <= d->wlog_slots && n_slots * 8 < dirty_bytes) {
            // mutation HETM_FAULT_SKIP_ROLLBACK: the first 1/8 of the write set (a chunk's worth of
            // state, "skip rollback of one chunk") is not rolled back
            const uint64_t skip = (d->fault & HETM_FAULT_SKIP_ROLLBACK) ? (n_slots / 8) & ~1ull : 0;
            e = launch_wlog_restore(d->d_cells, d->d_shadow, d->d_wlog + skip, n_slots - skip, d->W, d->geom,
                                    d->s_merge);
        }
        else
            e = launch_dirty_chunks(d->d_shadow, d->d_cells, d->W, d->d_chunk, d->chunk_bits, d->chunk_shift, false,
                                    d->geom, d->s_merge);
        if (e != cudaSuccess) return fail(d, e, "restore(rollback)");
        if ((rc = ensure_restore(d, std::max<uint64_t>(d->arena_n, d->recv_applied ? d->recv_cap : 0)))) return rc;
        e = launch_rollback_reapply(d->view(), d->d_shadow, round_logs(d), d->d_ctr, apply_queue(d, d->arena_n), d->geom,
                                    d->s_merge);
        if (e != cudaSuccess) return fail(d, e, "rollback_reapply");
        d->record(HETM_D2D, HETM_TAG_ROLLBACK, dirty_bytes);
        s.bytes_d2d = dirty_bytes;
        CK(d, cudaEventRecord(d->ev_shadow, d->s_merge));
    } else {
        if (!host) return HETM_ERR_INVALID_ARG;
        // Basic: host state copied over the device's dirty chunks
        if ((rc = ensure_stage(d, d->W))) return rc;
        for (auto& r : ranges) {
            CK(d, cudaMemcpyAsync(d->d_stage + r.first, host + r.first, r.second * 8, cudaMemcpyHostToDevice,
                                  d->s_merge));
            d->record(HETM_H2D, HETM_TAG_ROLLBACK, r.second * 8);
        }
        cudaError_t e = launch_dirty_chunks(d->d_stage, d->d_cells, d->W, d->d_chunk, d->chunk_bits, d->chunk_shift,
                                            false, d->geom, d->s_merge);
        if (e != cudaSuccess) return fail(d, e, "dirty_chunks(basic rollback)");
        s.bytes_h2d = dirty_bytes;
        if ((rc = refresh_shadow(d, true, dirty_bytes))) return rc;
    }
    CK(d, cudaStreamSynchronize(d->s_merge));
    s.dirty_chunks = nd;
    s.transfers = ranges.size();
    s.ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    if (st) *st = s;
    return HETM_OK;
}

int hetm_dev_merge_abort_host(hetm_dev* d, uint64_t* host, const uint64_t* snapshot, hetm_merge_stats* st) {
    NvtxRange nvtx_range("hetm.mergeAbortHost");
    if (!d || !host || !snapshot) return HETM_ERR_INVALID_ARG;
    auto t0 = std::chrono::steady_clock::now();
    std::lock_guard<std::mutex> g(d->mu);
    cancel_prepare(d);
    d->intake_open = false;
    if (d->round_applied) return HETM_ERR_STATE;  // FavorDevice validation is validate-only
    int rc = wait_round_work(d, d->s_merge);
    if (rc) return rc;
    CK(d, cudaStreamSynchronize(d->s_exec));
    CK(d, cudaStreamSynchronize(d->s_val));
    if (d->pool) d->pool->wait();  // a previous delta merge may still be landing in host_replica
    if (d->d2h_pending) CK(d, cudaStreamSynchronize(d->s_d2h));
    // hostReplica restored from the round-start snapshot
    std::memcpy(host, snapshot, d->W * 8);
    std::vector<std::pair<uint64_t, uint64_t>> ranges;
    uint64_t nd = 0;
    if ((rc = dirty_ranges(d, ranges, &nd))) return rc;
    uint64_t dirty_bytes = 0;
    for (auto& r : ranges) dirty_bytes += r.second * 8;
    const uint64_t* src = d->d_shadow;
    if (d->d_shadow) {
        if ((rc = refresh_shadow(d, false, dirty_bytes))) return rc;
    } else {
        if ((rc = ensure_stage(d, d->W))) return rc;
        cudaError_t e = launch_dirty_chunks(d->d_stage, d->d_cells, d->W, d->d_chunk, d->chunk_bits, d->chunk_shift,
                                            true, d->geom, d->s_merge);
        if (e != cudaSuccess) return fail(d, e, "dirty_chunks(stage)");
        CK(d, cudaEventRecord(d->ev_shadow, d->s_merge));
        src = d->d_stage;
    }
    CK(d, cudaStreamWaitEvent(d->s_d2h, d->ev_shadow, 0));
    for (auto& r : ranges) {
        CK(d, cudaMemcpyAsync(host + r.first, src + r.first, r.second * 8, cudaMemcpyDeviceToHost, d->s_d2h));
        d->record(HETM_D2H, HETM_TAG_MERGE, r.second * 8);
    }
    CK(d, cudaEventRecord(d->ev_d2h, d->s_d2h));
    CK(d, cudaStreamSynchronize(d->s_d2h));
    d->d2h_pending = false;
    // The discarded host log is dropped from the arena: nothing to re-apply.
    d->deferred.clear();
    if (st) {
        std::memset(st, 0, sizeof(*st));
        st->dirty_chunks = nd;
        st->transfers = ranges.size();
        st->bytes_d2h = dirty_bytes;
        st->ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    }
    return HETM_OK;
}

int hetm_dev_merge_wait(hetm_dev* d) {
    if (!d) return HETM_ERR_INVALID_ARG;
    if (d->pool) d->pool->wait();
    CK(d, cudaStreamSynchronize(d->s_merge));
    CK(d, cudaStreamSynchronize(d->s_d2h));
    d->d2h_pending = false;
    return HETM_OK;
}

int hetm_dev_clear_round(hetm_dev* d, uint32_t flags) {
    NvtxRange nvtx_range("hetm.clearRound");
    if (!d) return HETM_ERR_INVALID_ARG;
    std::lock_guard<std::mutex> g(d->mu);
    cancel_prepare(d);  // staged but never merged: not part of the replica
    int rc = wait_round_work(d, d->s_merge);
    if (rc) return rc;
    if (!(flags & HETM_CLEAR_ASYNC)) {
        CK(d, cudaStreamSynchronize(d->s_val));
        CK(d, cudaStreamSynchronize(d->s_exec));
    }
    // one kernel behind the round's work on s_merge (wait_round_work above);
    // the next round's work waits for ev_round
    cudaStream_t s = d->s_merge;
    {
        cudaError_t e = launch_clear_round(d->d_rs, d->d_ws, d->rs_words, d->d_chunk, d->chunk_words, d->d_ctr,
                                           (flags & HETM_CLEAR_RESET_TS) ? 1 : 0, d->geom, s);
        if (e != cudaSuccess) return fail(d, e, "clear_round");
    }
    if (flags & HETM_CLEAR_RESET_TS) {
        cudaError_t er = launch_reset_ts(d->d_cells, d->W, d->geom, s);
        if (er != cudaSuccess) return fail(d, er, "reset_ts");
    }
    CK(d, cudaEventRecord(d->ev_round, s));
    if (!(flags & HETM_CLEAR_ASYNC)) d->h_ctr->conflict = 0;
    d->arena_n = 0;
    d->ev_lo = 0;
    d->ev_pending = 0;
    d->sources.clear();
    d->recv_applied = 0;
    d->merge_staged = false;
    d->round_versioned = true;
    d->staged.active = false;
    d->deferred.clear();
    d->deferred_final = false;
    d->round_applied = false;
    d->round_tx = 0;
    d->intake_open = true;
    return HETM_OK;
}

// --------------------------------------------------------- transfer log
int hetm_dev_transfer_count(hetm_dev* d, uint64_t* n) {
    if (!d || !n) return HETM_ERR_INVALID_ARG;
    *n = d->xfer.size();
    return HETM_OK;
}

int hetm_dev_transfer_log(hetm_dev* d, hetm_transfer_record* out, uint64_t max, uint64_t* n) {
    if (!d || !n || (!out && max)) return HETM_ERR_INVALID_ARG;
    const uint64_t k = std::min<uint64_t>(max, d->xfer.size());
    std::copy(d->xfer.begin(), d->xfer.begin() + (ptrdiff_t)k, out);
    *n = d->xfer.size();
    return HETM_OK;
}

int hetm_dev_clear_transfer_log(hetm_dev* d) {
    if (!d) return HETM_ERR_INVALID_ARG;
    d->xfer.clear();
    return HETM_OK;
}

// --------------------------------------------------- device-resident entries
int hetm_dev_execute_batch_dptr(hetm_dev* d, int kernel_id, const void* d_inputs, uint64_t n_tx, uint64_t* d_tickets,
                                void* stream) {
    if (!d || (n_tx && (!d_inputs || !d_tickets))) return HETM_ERR_INVALID_ARG;
    if (!d->kernels.count(kernel_id)) return HETM_ERR_KERNEL_NOT_REGISTERED;
    if (n_tx >= (1ull << 30)) return HETM_ERR_INVALID_SIZE;
    cudaStream_t s = stream ? static_cast<cudaStream_t>(stream) : d->s_exec;
    return enqueue_batch(d, kernel_id, d_inputs, n_tx, reinterpret_cast<unsigned long long*>(d_tickets), nullptr, s);
}

int hetm_dev_execute_batch_dptr_ex(hetm_dev* d, int kernel_id, const void* d_inputs, uint64_t n_tx,
                                   uint64_t* d_tickets, void* d_results, void* stream) {
    if (!d || (n_tx && (!d_inputs || !d_tickets))) return HETM_ERR_INVALID_ARG;
    if (!d->kernels.count(kernel_id)) return HETM_ERR_KERNEL_NOT_REGISTERED;
    if (n_tx >= (1ull << 30)) return HETM_ERR_INVALID_SIZE;
    if (d_results && kernel_id != HETM_KERNEL_CACHE) return HETM_ERR_INVALID_SIZE;
    cudaStream_t s = stream ? static_cast<cudaStream_t>(stream) : d->s_exec;
    bool hot = false;
    if (kernel_id == HETM_KERNEL_BANK && d->schedule == HETM_SCHED_AUTO && n_tx) {
        // AUTO without a host view of the inputs: follow the estimate of an earlier
        // device batch (written to mapped host memory, read without a sync) and
        // estimate this one on a side stream for the next.
        if (!d->h_hot) {
            CK(d, cudaHostAlloc((void**)&d->h_hot, 64, cudaHostAllocMapped));
            *d->h_hot = 0;
            CK(d, cudaHostGetDevicePointer((void**)&d->d_hot, d->h_hot, 0));
            CK(d, cudaStreamCreateWithFlags(&d->s_est, cudaStreamNonBlocking));
            CK(d, cudaEventCreateWithFlags(&d->ev_est, cudaEventDisableTiming));
        }
        const uint32_t last = *reinterpret_cast<volatile uint32_t*>(d->h_hot);
        const bool feedback = d->auto_scan_left > 0;
        if (feedback) --d->auto_scan_left;
        hot = feedback || hot_chain(last, n_tx, bank_hot_estimate_sample(n_tx), sched_chain());
    }
    d->dptr_feedback_n = kernel_id == HETM_KERNEL_BANK && d->schedule == HETM_SCHED_AUTO && !hot ? n_tx : 0;
    if (int rc = enqueue_batch(d, kernel_id, d_inputs, n_tx, reinterpret_cast<unsigned long long*>(d_tickets),
                               d_results, s, true, nullptr, hot))
        return rc;
    if (d->s_est && kernel_id == HETM_KERNEL_BANK && d->schedule == HETM_SCHED_AUTO && n_tx) {
        // the estimate for the next batch starts once this batch's kernels are done:
        // its CTA (128 KiB of shared memory) must never hold an SM the batch's
        // persistent CTAs need (it overlaps the validation phase instead)
        // The sampled records are copied into a handle-owned buffer on the batch's
        // stream first (S strided records, 48 KiB): the caller may free or reuse
        // d_inputs once that stream is done, while the estimate still runs on s_est.
        const uint64_t S = bank_hot_estimate_sample(n_tx), stride = n_tx / S;
        if (!d->d_est_in) {
            if (int rc = dev_alloc(d, (void**)&d->d_est_in, bank_hot_estimate_sample(~0ull) * sizeof(hetm_bank_tx)))
                return rc;
        }
        CK(d, cudaMemcpy2DAsync(d->d_est_in, sizeof(hetm_bank_tx), d_inputs, stride * sizeof(hetm_bank_tx),
                                sizeof(hetm_bank_tx), S, cudaMemcpyDeviceToDevice, s));
        CK(d, cudaEventRecord(d->ev_est, s));
        CK(d, cudaStreamWaitEvent(d->s_est, d->ev_est, 0));
        cudaError_t e = launch_bank_hot_estimate(d->d_est_in, S, d->d_hot, d->s_est);
        if (e != cudaSuccess) return fail(d, e, "hot_estimate");
    }
    return HETM_OK;
}

int hetm_dev_set_cache_geometry(hetm_dev* d, uint64_t base_word, uint64_t n_sets) {
    if (!d) return HETM_ERR_INVALID_ARG;
    if (n_sets < 2 || (n_sets & (n_sets - 1))) return HETM_ERR_INVALID_SIZE;
    if (base_word < d->base || base_word - d->base + n_sets * HETM_CACHE_SET_WORDS > d->W)
        return HETM_ERR_OUT_OF_BOUNDS;
    d->cache.base_local = base_word - d->base;
    d->cache.n_sets = n_sets;
    return HETM_OK;
}

uint64_t hetm_cache_hash(uint64_t key0, uint64_t key1) { return cache_hash(key0, key1); }
uint64_t hetm_cache_set_of(uint64_t key0, uint64_t key1, uint64_t n_sets) {
    return n_sets >= 2 ? cache_set_of(key0, key1, n_sets) : 0;
}

int hetm_dev_validate_dptr(hetm_dev* d, const hetm_log_entry* d_entries, uint64_t n, int mode, void* stream) {
    if (!d || (n && !d_entries)) return HETM_ERR_INVALID_ARG;
    const bool retain = (mode & HETM_RETAIN) != 0;
    mode &= ~HETM_RETAIN;
    if (mode != HETM_APPLY && mode != HETM_VALIDATE_ONLY) return HETM_ERR_INVALID_ARG;
    if (d->merge_staged) return HETM_ERR_ROUND_CLOSED;  // the merge has started
    cudaStream_t s = stream ? static_cast<cudaStream_t>(stream) : d->s_val;
    if (mode == HETM_APPLY)
        if (int rc = ensure_restore(d, n)) return rc;
    if (retain) {  // the entries join the round's arena (D2D), so the shadow patch and the rollback see them
        std::lock_guard<std::mutex> g(d->mu);
        if (int rc = ensure_arena(d, d->arena_n + n)) return rc;
    }
    CK(d, cudaStreamWaitEvent(s, d->ev_round, 0));
    if (retain && n) {
        hetm_log_entry* dst = d->d_arena + d->arena_n;
        CK(d, cudaMemcpyAsync(dst, d_entries, n * sizeof(hetm_log_entry), cudaMemcpyDeviceToDevice, s));
        d->record(HETM_D2D, HETM_TAG_LOG, n * sizeof(hetm_log_entry));
        d_entries = dst;
        d->arena_n += n;
        d->ev_lo = d->arena_n;
    }
    if (mode == HETM_APPLY) {
        CK(d, cudaStreamWaitEvent(s, d->ev_exec, 0));
        d->round_applied = true;
        if (!retain) d->shadow_synced = false;  // not in the arena: the next shadow refresh is a full copy
    }
    cudaError_t e = timed_validate(d, d_entries, n, mode == HETM_APPLY, s);
    if (e != cudaSuccess) return fail(d, e, "validate_dptr");
    return join_val(d, s);
}

int hetm_dev_read_counters(hetm_dev* d, int* conflict, hetm_batch_stats* last) {
    if (!d) return HETM_ERR_INVALID_ARG;
    CK(d, cudaDeviceSynchronize());
    int rc = read_counters(d);
    if (rc) return rc;
    if (conflict) *conflict = d->h_ctr->conflict ? 1 : 0;
    if (last) {
        std::memset(last, 0, sizeof(*last));
        last->committed = d->h_ctr->committed;
        last->aborts = d->h_ctr->aborts;
        last->retried = d->h_ctr->retried;
        last->livelocked = d->h_ctr->livelocked;
        last->ticket_end = d->h_ctr->ticket;
    }
    if (d->h_ctr->oob) return HETM_ERR_OUT_OF_BOUNDS;
    return HETM_OK;
}

int hetm_dev_route_log_dptr(hetm_dev* d, const hetm_log_entry* d_in, uint64_t n, uint32_t n_shards,
                            uint64_t shard_words, hetm_log_entry* d_out, uint64_t* d_counts, void* stream) {
    if (!d || (n && (!d_in || !d_out)) || !d_counts) return HETM_ERR_INVALID_ARG;
    if (n_shards == 0 || n_shards > 64 || shard_words == 0) return HETM_ERR_CONFIG;
    const size_t need = route_log_scratch_bytes(n, n_shards, d->geom);
    if (need > d->route_cap) {
        if (d->d_route) { CK(d, cudaDeviceSynchronize()); cudaFree(d->d_route); }
        int rc = dev_alloc(d, &d->d_route, need);
        if (rc) return rc;
        d->route_cap = need;
    }
    cudaStream_t s = stream ? static_cast<cudaStream_t>(stream) : d->s_val;
    cudaError_t e = launch_route_log(d_in, n, n_shards, shard_words, d_out,
                                     reinterpret_cast<unsigned long long*>(d_counts), d->d_route, d->route_cap,
                                     d->geom, s);
    if (e != cudaSuccess) return fail(d, e, "route_log");
    return HETM_OK;
}

int hetm_dev_recv_arena(hetm_dev* d, uint32_t n_shards, uint64_t cap, void** d_entries, void** d_counts) {
    if (!d || !d_entries || !d_counts || n_shards == 0 || n_shards > 64 || cap == 0) return HETM_ERR_INVALID_ARG;
    if (n_shards != d->recv_shards || cap != d->recv_cap) {
        int rc = sync_all(d);
        if (rc) return rc;
        if (d->d_recv) { cudaFree(d->d_recv); d->bytes_alloc -= 2 * d->recv_shards * d->recv_cap * sizeof(hetm_log_entry); }
        if (d->d_recv_counts) { cudaFree(d->d_recv_counts); d->bytes_alloc -= 128 * 8; }
        d->d_recv = nullptr;
        d->d_recv_counts = nullptr;
        // two arenas (round parity): a sender may route round r+1 while this owner still applies round r
        if ((rc = dev_alloc(d, (void**)&d->d_recv, 2 * (size_t)n_shards * cap * sizeof(hetm_log_entry)))) return rc;
        if ((rc = dev_alloc(d, (void**)&d->d_recv_counts, 128 * 8))) return rc;
        CK(d, cudaMemset(d->d_recv_counts, 0, 128 * 8));
        d->recv_shards = n_shards;
        d->recv_cap = cap;
    }
    *d_entries = d->d_recv;
    *d_counts = d->d_recv_counts;
    return HETM_OK;
}

int hetm_dev_route_to_peers_dptr(hetm_dev* d, const hetm_log_entry* d_in, uint64_t n, uint32_t n_shards,
                                 uint64_t shard_words, uint32_t my_shard, uint64_t cap, uint32_t parity,
                                 void* const* peer_entries, void* const* peer_counts, void* stream) {
    NvtxRange nvtx_range("hetm.routeToPeers");
    if (!d || (n && !d_in) || !peer_entries || !peer_counts) return HETM_ERR_INVALID_ARG;
    if (n_shards == 0 || n_shards > 64 || shard_words == 0 || my_shard >= n_shards) return HETM_ERR_CONFIG;
    if (n > cap) return HETM_ERR_INVALID_SIZE;
    int rc;
    const size_t need = route_log_scratch_bytes(n, n_shards, d->geom);
    if (need > d->route_cap) {
        if (d->d_route) { CK(d, cudaDeviceSynchronize()); cudaFree(d->d_route); }
        if ((rc = dev_alloc(d, &d->d_route, need))) return rc;
        d->route_cap = need;
    }
    if (!d->d_peer_ptrs) {
        if ((rc = dev_alloc(d, (void**)&d->d_peer_ptrs, 2 * 128 * sizeof(void*)))) return rc;
        if ((rc = dev_alloc(d, (void**)&d->d_peer_totals, 64 * 8))) return rc;
    }
    const uint32_t par = parity & 1;
    std::array<void*, 128> table{};
    for (uint32_t s = 0; s < n_shards; ++s) {  // this round's arena / count block of every owner
        table[s] = static_cast<hetm_log_entry*>(peer_entries[s]) + (uint64_t)par * n_shards * cap;
        table[64 + s] = static_cast<unsigned long long*>(peer_counts[s]) + par * 64;
    }
    cudaStream_t s = stream ? static_cast<cudaStream_t>(stream) : d->s_val;
    void** dtab = d->d_peer_ptrs + par * 128;
    // the IPC-opened peer pointers do not change between rounds: each parity's
    // device table is uploaded once (again only if the peers change), so a
    // round's routing never waits on the host
    if (!d->peer_table_ok[par] || d->peer_table[par] != table) {
        CK(d, cudaStreamSynchronize(s));  // a launch of two rounds ago may still read this parity's table
        CK(d, cudaMemcpy(dtab, table.data(), sizeof(void*) * 128, cudaMemcpyHostToDevice));
        d->peer_table[par] = table;
        d->peer_table_ok[par] = true;
    }
    cudaError_t e = launch_route_to_peers(d_in, n, n_shards, shard_words, my_shard, cap,
                                          reinterpret_cast<hetm_log_entry* const*>(dtab),
                                          reinterpret_cast<unsigned long long* const*>(dtab + 64),
                                          d->d_peer_totals, d->d_route, d->route_cap, d->geom, s);
    if (e != cudaSuccess) return fail(d, e, "route_to_peers");
    return HETM_OK;
}

int hetm_dev_apply_received(hetm_dev* d, uint32_t parity, int mode, uint64_t* n_out, void* stream) {
    NvtxRange nvtx_range("hetm.applyReceived");
    if (!d || !d->d_recv) return HETM_ERR_INVALID_ARG;
    if (mode != HETM_APPLY && mode != HETM_VALIDATE_ONLY) return HETM_ERR_INVALID_ARG;
    cudaStream_t s = stream ? static_cast<cudaStream_t>(stream) : d->s_val;
    const uint64_t p = parity & 1;
    const hetm_log_entry* arena = d->d_recv + p * d->recv_shards * d->recv_cap;
    const unsigned long long* counts = d->d_recv_counts + p * 64;
    if (mode == HETM_APPLY)
        if (int rc = ensure_restore(d, d->recv_cap)) return rc;
    CK(d, cudaStreamWaitEvent(s, d->ev_round, 0));
    if (mode == HETM_APPLY) {
        CK(d, cudaStreamWaitEvent(s, d->ev_exec, 0));
        d->round_applied = true;
        // the regions stay in the receive arena until the next round of this
        // parity: the shadow patch and the optimized rollback read them there
        d->recv_applied |= 1u << p;
    }
    // one launch over every received region; the counts stay on the device
    cudaEvent_t t0 = nullptr, t1 = nullptr;
    if (d->timing) {
        t0 = d->tev();
        t1 = d->tev();
        cudaEventRecord(t0, s);
    }
    const cudaError_t e = launch_validate_regions(d->view(), arena, counts, d->recv_shards, d->recv_cap,
                                                  mode == HETM_APPLY ? 1 : 0, d->d_ctr,
                                                  mode == HETM_APPLY ? apply_queue(d, (uint64_t)d->recv_shards * d->recv_cap)
                                                                     : RestoreQueue{d->d_restore, d->restore_cap},
                                                  d->geom, s);
    if (d->timing) {
        cudaEventRecord(t1, s);
        d->tpairs[1].emplace_back(t0, t1);
    }
    if (e != cudaSuccess) return fail(d, e, "validate_regions");
    if (int rc = join_val(d, s)) return rc;
    if (n_out) {  // optional: the entry count needs a host round trip
        unsigned long long c[64] = {};
        CK(d, cudaMemcpyAsync(c, counts, d->recv_shards * 8, cudaMemcpyDeviceToHost, s));
        CK(d, cudaStreamSynchronize(s));
        uint64_t total = 0;
        for (uint32_t r = 0; r < d->recv_shards; ++r) total += std::min<uint64_t>(c[r], d->recv_cap);
        *n_out = total;
    }
    return HETM_OK;
}

int hetm_ipc_get_handle(void* dptr, void* handle64) {
    if (!dptr || !handle64) return HETM_ERR_INVALID_ARG;
    cudaIpcMemHandle_t h;
    const cudaError_t e = cudaIpcGetMemHandle(&h, dptr);
    if (e != cudaSuccess) {
        cudaGetLastError();
        return HETM_ERR_CUDA;
    }
    static_assert(sizeof(h) == 64, "IPC handle size");
    std::memcpy(handle64, &h, 64);
    return HETM_OK;
}

int hetm_ipc_open_handle(const void* handle64, void** dptr) {
    if (!handle64 || !dptr) return HETM_ERR_INVALID_ARG;
    cudaIpcMemHandle_t h;
    std::memcpy(&h, handle64, 64);
    const cudaError_t e = cudaIpcOpenMemHandle(dptr, h, cudaIpcMemLazyEnablePeerAccess);
    if (e != cudaSuccess) {
        cudaGetLastError();
        *dptr = nullptr;
        return HETM_ERR_CUDA;
    }
    return HETM_OK;
}

int hetm_ipc_close(void* dptr) {
    if (!dptr) return HETM_ERR_INVALID_ARG;
    cudaIpcCloseMemHandle(dptr);
    return HETM_OK;
}

int hetm_enable_peer_access(int device, int peer) {
    int can = 0;
    if (cudaDeviceCanAccessPeer(&can, device, peer) != cudaSuccess || !can) {
        cudaGetLastError();
        return HETM_ERR_CUDA;
    }
    int cur = 0;
    cudaGetDevice(&cur);
    cudaSetDevice(device);
    const cudaError_t e = cudaDeviceEnablePeerAccess(peer, 0);
    cudaSetDevice(cur);
    if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled) {
        cudaGetLastError();
        return HETM_ERR_CUDA;
    }
    cudaGetLastError();
    return HETM_OK;
}

int hetm_dev_trace_next_batch(hetm_dev* d, uint64_t* out_records) {
    if (!d || !out_records) return HETM_ERR_INVALID_ARG;
    std::lock_guard<std::mutex> g(d->mu);
    d->trace_out = out_records;
    return HETM_OK;
}

int hetm_dev_set_schedule(hetm_dev* d, int mode) {
    if (!d || mode < HETM_SCHED_OPTIMISTIC || mode > HETM_SCHED_AUTO) return HETM_ERR_INVALID_ARG;
    std::lock_guard<std::mutex> g(d->mu);
    d->schedule = mode;
    return HETM_OK;
}

int hetm_dev_set_fault(hetm_dev* d, uint32_t flags) {
    if (!d || (flags & ~(uint32_t)HETM_FAULT_ALL)) return HETM_ERR_INVALID_ARG;
    std::lock_guard<std::mutex> g(d->mu);
    if ((flags & HETM_FAULT_SKIP_RS) && !d->d_rs_zero) {
        if (int rc = dev_alloc(d, (void**)&d->d_rs_zero, d->rs_words * 8)) return rc;
        CK(d, cudaMemset(d->d_rs_zero, 0, d->rs_words * 8));
    }
    d->fault = flags;
    return HETM_OK;
}

int hetm_dev_stream_handle(hetm_dev* d, int which, void** stream) {
    if (!d || !stream) return HETM_ERR_INVALID_ARG;
    cudaStream_t s[5] = {d->s_exec, d->s_copy, d->s_val, d->s_merge, d->s_d2h};
    if (which < 0 || which > 4) return HETM_ERR_INVALID_ARG;
    *stream = s[which];
    return HETM_OK;
}

int hetm_dev_debug_words(hetm_dev* d, uint64_t* out, uint64_t n) {
    if (!d || !out || n > 18) return HETM_ERR_INVALID_ARG;
    int rc = sync_all(d);
    if (rc) return rc;
    if ((rc = read_counters(d))) return rc;
    for (uint64_t i = 0; i < n; ++i) out[i] = d->h_ctr->pad[i];
    return HETM_OK;
}

int hetm_dev_set_timing(hetm_dev* d, int on) {
    if (!d) return HETM_ERR_INVALID_ARG;
    d->timing = on != 0;
    return HETM_OK;
}

int hetm_dev_timing(hetm_dev* d, int which, double* total_ms, uint64_t* count) {
    if (!d || which < 0 || which > 2) return HETM_ERR_INVALID_ARG;
    double tot = 0;
    uint64_t c = 0;
    for (auto& pr : d->tpairs[which]) {
        CK(d, cudaEventSynchronize(pr.second));
        float ms = 0.f;
        CK(d, cudaEventElapsedTime(&ms, pr.first, pr.second));
        tot += ms;
        ++c;
        d->tpool.push_back(pr.first);
        d->tpool.push_back(pr.second);
    }
    d->tpairs[which].clear();
    if (total_ms) *total_ms = tot;
    if (count) *count = c;
    return HETM_OK;
}

int hetm_dev_flush_l2(hetm_dev* d, void* stream) {
    if (!d) return HETM_ERR_INVALID_ARG;
    if (!d->d_flush) {
        d->flush_bytes = std::max<uint64_t>(2 * d->l2_bytes, 256ull << 20);
        int rc = dev_alloc(d, &d->d_flush, d->flush_bytes);
        if (rc) return rc;
    }
    cudaStream_t s = stream ? static_cast<cudaStream_t>(stream) : d->s_exec;
    CK(d, cudaMemsetAsync(d->d_flush, (int)(++d->flush_gen & 0xff), d->flush_bytes, s));
    return HETM_OK;
}

// ------------------------------------------------------------------ host side
// Large pinned host buffers (host replica, delta landing zones) are backed by
// 2 MiB transparent huge pages when the kernel allows it (madvise mode): the
// delta merge scatters ~10^6 words per round into the host replica, and 4 KiB
// pages make every write a TLB miss.
namespace {
std::mutex g_host_mu;
std::map<void*, std::pair<void*, size_t>> g_host_maps;  // aligned ptr -> (mmap base, mmap length)
constexpr size_t kHuge = 2ull << 20;
}  // namespace

int hetm_host_alloc(uint64_t bytes, void** p) {
    if (!p) return HETM_ERR_INVALID_ARG;
    *p = nullptr;
    if (bytes >= 2 * kHuge) {
        const size_t len = (bytes + kHuge - 1) / kHuge * kHuge + kHuge;
        void* base = mmap(nullptr, len, PROT_READ | PROT_WRITE, MAP_PRIVATE | MAP_ANONYMOUS, -1, 0);
        if (base != MAP_FAILED) {
            void* al = reinterpret_cast<void*>((reinterpret_cast<uintptr_t>(base) + kHuge - 1) & ~(uintptr_t)(kHuge - 1));
            madvise(al, len - kHuge, MADV_HUGEPAGE);
            const cudaError_t e = cudaHostRegister(al, len - kHuge, cudaHostRegisterPortable);
            if (e == cudaSuccess) {
                std::lock_guard<std::mutex> g(g_host_mu);
                g_host_maps[al] = {base, len};
                *p = al;
                return HETM_OK;
            }
            cudaGetLastError();
            munmap(base, len);
            if (e == cudaErrorNoDevice || e == cudaErrorInsufficientDriver) return HETM_ERR_NO_DEVICE;
        }
    }
    cudaError_t e = cudaHostAlloc(p, bytes ? bytes : 8, cudaHostAllocPortable);
    if (e != cudaSuccess) {
        cudaGetLastError();
        *p = nullptr;
        return e == cudaErrorNoDevice || e == cudaErrorInsufficientDriver ? HETM_ERR_NO_DEVICE : HETM_ERR_CUDA;
    }
    return HETM_OK;
}

int hetm_host_free(void* p) {
    if (!p) return HETM_OK;
    {
        std::lock_guard<std::mutex> g(g_host_mu);
        auto it = g_host_maps.find(p);
        if (it != g_host_maps.end()) {
            cudaHostUnregister(p);
            munmap(it->second.first, it->second.second);
            g_host_maps.erase(it);
            return HETM_OK;
        }
    }
    cudaFreeHost(p);
    return HETM_OK;
}

int hetm_host_register(void* p, uint64_t bytes) {
    if (!p) return HETM_ERR_INVALID_ARG;
    cudaError_t e = cudaHostRegister(p, bytes, cudaHostRegisterPortable);
    if (e != cudaSuccess) {
        cudaGetLastError();
        return e == cudaErrorNoDevice || e == cudaErrorInsufficientDriver ? HETM_ERR_NO_DEVICE : HETM_ERR_CUDA;
    }
    return HETM_OK;
}

int hetm_host_unregister(void* p) {
    if (!p) return HETM_ERR_INVALID_ARG;
    cudaHostUnregister(p);
    return HETM_OK;
}

}  // extern "C"
