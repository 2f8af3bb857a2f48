// kernels.h — host-callable launchers for the sm_100a kernels (internal).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "hetm_b200/capi.h"

namespace hetm_b200 {

struct DevCounters;
struct ShardView;
struct Cell;
struct CacheGeom;

// One merge delta record: local word index + value (16 B, DMA'd to the host).
// Merge delta records, struct of arrays (12 B per record on the wire): the
// shard-local word (< 2^32; ~0u = empty slot) and its value.
struct DeltaBuf {
    uint32_t* loc;
    uint64_t* val;
};

struct LaunchGeom {
    int sm_count;
    int max_blocks_tx;    // resident blocks per SM for the batch kernels
    int max_blocks_val;   // resident blocks per SM for the validation kernels
};

// guest-stm-batch: one launch executes a whole batch.
cudaError_t launch_bank_batch(const ShardView& v, const hetm_bank_tx* d_in, uint64_t n, unsigned long long* d_tickets,
                              DevCounters* ctr, uint32_t max_attempts, const LaunchGeom& g, cudaStream_t s);
cudaError_t launch_cache_batch(const ShardView& v, const CacheGeom& cg, const hetm_cache_tx* d_in, uint64_t n,
                               unsigned long long* d_tickets, hetm_cache_result* d_res, DevCounters* ctr,
                               uint32_t max_attempts, const LaunchGeom& g, cudaStream_t s);
cudaError_t launch_rw_batch(const ShardView& v, const hetm_rw_tx* d_in, uint64_t n, unsigned long long* d_tickets,
                            DevCounters* ctr, uint32_t max_attempts, const LaunchGeom& g, cudaStream_t s);

// engine.validateChunk over n log entries (apply: pass A + pass B).
// Apply-mode launches of one handle must be stream-ordered (they share the
// restore queue and rely on the previous launch's stores being complete).
// Restore queue of the apply kernel: indices of entries whose value store raced
// with another entry of the round; overflow (> cap) falls back to a full
// winner pass over the launch.  The handle sizes cap to the launch (n/4).
struct RestoreQueue {
    unsigned long long* idx;
    uint64_t cap;
    int amax = 0;  // apply form of the launch: 0 exchange (no restore pass), 1 atomicMax + restore (hot logs)
};
cudaError_t launch_blind_apply(const ShardView& v, const hetm_log_entry* d_log, uint64_t n, DevCounters* ctr,
                               const LaunchGeom& g, cudaStream_t s);  // fault injection only
cudaError_t launch_validate(const ShardView& v, const hetm_log_entry* d_log, uint64_t n, int apply,
                            DevCounters* ctr, RestoreQueue rq, const LaunchGeom& g, cudaStream_t s);
// The round's host log on one device: the arena (flat, in arrival order) and
// the peer-arena region sets it received this round (multi-GPU exchange).
struct RoundLogRegions {
    const hetm_log_entry* base;
    const unsigned long long* counts;  // device counts of the regions
    uint32_t n_regions;
    uint64_t cap;
};
struct RoundLogs {
    const hetm_log_entry* flat;
    uint64_t n;
    RoundLogRegions region[2];  // one per round parity applied this round
    uint32_t n_regions_sets;
};
// Optimized rollback: untag the logged words, re-apply the round logs, copy them to shadow.
cudaError_t launch_rollback_reapply(const ShardView& v, uint64_t* shadow, const RoundLogs& logs, DevCounters* ctr,
                                    RestoreQueue rq, const LaunchGeom& g, cudaStream_t s);
// Literal TS reset: every TS word becomes an unlocked word.
cudaError_t launch_reset_ts(Cell* cells, uint64_t size_words, const LaunchGeom& g, cudaStream_t s);
// Validate/apply the received regions of a peer arena (counts on the device; no host sync).
cudaError_t launch_validate_regions(const ShardView& v, const hetm_log_entry* d_base, const unsigned long long* d_counts,
                                    uint32_t n_regions, uint64_t cap, int apply, DevCounters* ctr,
                                    RestoreQueue rq, const LaunchGeom& g, cudaStream_t s);
// Round boundary: ts_floor = max(ts_floor, round_max_ts) (0 with reset_ts), round_max_ts = 0.
// Winner store of the round's log: value of the entry whose ts equals the
// cell's TS goes to dst[addr] (plain array) or, with dst == nullptr, to the
// cell's value (rollback / shadow patch).
cudaError_t launch_winner_apply(Cell* cells, uint64_t* dst, uint64_t base, uint64_t size_words,
                                const hetm_log_entry* d_log, uint64_t n, const LaunchGeom& g, cudaStream_t s,
                                const DevCounters* gate = nullptr);
// The same over received peer-arena regions (counts on the device).
cudaError_t launch_winner_regions(Cell* cells, uint64_t* dst, uint64_t base, uint64_t size_words,
                                  const hetm_log_entry* d_base, const unsigned long long* d_counts,
                                  uint32_t n_regions, uint64_t cap, const LaunchGeom& g, cudaStream_t s,
                                  const DevCounters* gate = nullptr);
// Word-cell <-> plain word conversions (cells.cu).
cudaError_t launch_gather_range(uint64_t* dst, const Cell* cells, uint64_t lo, uint64_t n, const LaunchGeom& g,
                                cudaStream_t s);
cudaError_t launch_scatter_range(Cell* cells, const uint64_t* src, uint64_t lo, uint64_t n, const LaunchGeom& g,
                                 cudaStream_t s);
// bits == nullptr: every chunk.  to_plain: plain[w] = cells[w].value, else the reverse.
cudaError_t launch_dirty_chunks(uint64_t* plain, Cell* cells, uint64_t size_words, const unsigned long long* bits,
                                uint64_t n_chunks, uint32_t chunk_shift, bool to_plain, const LaunchGeom& g,
                                cudaStream_t s);
// Write-set log -> compact delta in two hand-written passes (cells.cu): claim
// (dedup through a W-bit claim bitmap, unique-word list, address-bucket
// counts), then emit ({word, value} records grouped by bucket, devShadow
// refreshed when shadow != nullptr, claim words cleared).  The record count
// is *n_uniq on the device.
constexpr uint32_t kDeltaBucketBits = 8;  // 256 address ranges (4 MiB of a 1 GiB replica each)
constexpr int kDeltaBuckets = 1 << kDeltaBucketBits;
struct DeltaScratch {
    unsigned long long* claim;      // ceil(W/64) words, all zero between stages
    uint32_t* uniq;                 // unique words (claim pass) / per-slot picked word or ~0u (pick pass)
    uint64_t* uniq_val;             // per-slot values (pick pass only)
    unsigned long long* n_uniq;     // [0] record count, [1] slot count (pick pass)
    uint32_t* bucket_cnt;           // kDeltaBuckets counts, then kDeltaBuckets cursors
    // bytes from n_uniq through the end of bucket_cnt when both live in one
    // allocation (one memset clears the stage's counters), else 0
    size_t counters_bytes = 0;
};
uint32_t delta_bucket_shift(uint64_t size_words);
cudaError_t launch_delta_claim(const uint32_t* wlog, uint64_t n, uint64_t size_words, const DeltaScratch& ds,
                               const LaunchGeom& g, cudaStream_t s, const DevCounters* gate = nullptr);
// Versioned replacement of the claim pass (rounds of bank / rw batches only):
// the slot whose ticket's commit version is still in the word's cell picks
// the word and its value (no claim bitmap, no atomics on the words).
cudaError_t launch_delta_pick(const uint32_t* wlog, uint64_t n, uint64_t size_words, const Cell* cells,
                              const DeltaScratch& ds, const LaunchGeom& g, cudaStream_t s, const DevCounters* ctr,
                              bool gated);
cudaError_t launch_delta_emit(uint64_t max_records, uint64_t size_words, const DeltaScratch& ds, const Cell* cells,
                              DeltaBuf out, uint64_t* shadow, const LaunchGeom& g, cudaStream_t s,
                              bool picked = false);
// Rollback of the device write set: cells[loc].value = shadow[loc] per log slot.
cudaError_t launch_wlog_restore(Cell* cells, const uint64_t* shadow, const uint32_t* wlog, uint64_t n,
                                uint64_t size_words, const LaunchGeom& g, cudaStream_t s);
// Zero-copy scatter of delta records into a device-accessible host buffer.
cudaError_t launch_delta_zc_scatter(uint64_t* host_dev, DeltaBuf d, uint64_t n, const LaunchGeom& g,
                                    cudaStream_t s);
// SCAN schedule of a bank batch (bank_sched.cu): sort + segmented scan, input
// order, no aborts; temp from bank_sched_temp_bytes.
size_t bank_sched_temp_bytes(uint64_t n, uint64_t size_words);
// Device-side hot-spot estimate: largest account count among
// bank_hot_estimate_sample(n) sampled transactions -> *out (mapped host word).
cudaError_t launch_bank_hot_estimate(const hetm_bank_tx* d_in, uint64_t n, uint32_t* out, cudaStream_t s);
uint64_t bank_hot_estimate_sample(uint64_t n);
// Captured CUDA graph of the untraced SCAN sequence (one per handle), rebuilt
// when the batch size or a buffer changes; nullptr launches kernel by kernel.
struct SchedGraph {
    cudaGraphExec_t exec = nullptr;
    cudaGraph_t graph = nullptr;  // kept: the exec's node handles refer to it
    cudaStream_t cap = nullptr;   // private capture stream
    cudaGraphNode_t keys_node = nullptr;
    cudaKernelNodeParams keys_params{};
    // owned copies of the keys kernel's arguments (the captured node's own
    // storage dies with the graph): its signature in bank_sched.cu
    struct KeysArgs {
        ShardView v;
        const void* in;
        uint64_t n;
        void *locs, *pay, *delta, *tickets;
        const void* first;
        void* ctr;
    } keys_args{};
    void* keys_ptrs[9] = {};
    uint64_t n = 0, wlog_slots = 0;
    void* temp = nullptr;
    const void* wlog = nullptr;
    const void* cells = nullptr;
    const void* ctr = nullptr;
};
cudaError_t launch_bank_sched(const ShardView& v, const hetm_bank_tx* d_in, uint64_t n, unsigned long long* d_tickets,
                              DevCounters* ctr, void* temp, size_t temp_bytes, const LaunchGeom& g, cudaStream_t s,
                              SchedGraph* graph = nullptr);
// SCAN schedule of a cache batch (cache_sched.cu): stable sort by set, one
// thread per set runs its transactions in input order; no locks, no aborts.
size_t cache_sched_temp_bytes(uint64_t n, uint64_t n_sets);
cudaError_t launch_cache_sched(const ShardView& v, const CacheGeom& cg, const hetm_cache_tx* d_in, uint64_t n,
                               unsigned long long* d_tickets, hetm_cache_result* d_res, DevCounters* ctr, void* temp,
                               size_t temp_bytes, const LaunchGeom& g, cudaStream_t s);
// devShadow[loc] = value for staged delta records (prepared merge).
cudaError_t launch_delta_to_shadow(uint64_t* shadow, DeltaBuf d, uint64_t n, const LaunchGeom& g, cudaStream_t s);
// dst[lo, hi) |= peers[k][lo, hi) for every peer bitmap (NVLink peer loads).
cudaError_t launch_or_peers(unsigned long long* dst, const unsigned long long* const* peers, uint32_t n_peers,
                            uint64_t lo, uint64_t hi, const LaunchGeom& g, cudaStream_t s);
// Asynchronous clearRound in one launch (bitmaps zeroed + round counters rolled).
cudaError_t launch_clear_round(unsigned long long* rs, unsigned long long* ws, uint64_t rs_words,
                               unsigned long long* chunk, uint64_t chunk_words, DevCounters* ctr, int reset_ts,
                               const LaunchGeom& g, cudaStream_t s);
// Popcount of n words into *out (device counter, accumulated).
cudaError_t launch_popcount(const unsigned long long* words, uint64_t n, unsigned long long* out, cudaStream_t s);
// OR src words into dst words.
cudaError_t launch_or_words(unsigned long long* dst, const unsigned long long* src, uint64_t n, cudaStream_t s);
// Shard router: stable partition of entries by owner = addr / shard_words.
cudaError_t launch_route_log(const hetm_log_entry* d_in, uint64_t n, uint32_t n_shards, uint64_t shard_words,
                             hetm_log_entry* d_out, unsigned long long* d_counts, void* d_scratch,
                             size_t scratch_bytes, const LaunchGeom& g, cudaStream_t s);
size_t route_log_scratch_bytes(uint64_t n, uint32_t n_shards, const LaunchGeom& g);
// Route + deliver: entries of shard s land in d_peer_out[s][my*cap ...], bucket sizes in
// d_peer_counts[s][my] (device arrays of n_shards pointers, peer/IPC pointers allowed).
cudaError_t launch_route_to_peers(const hetm_log_entry* d_in, uint64_t n, uint32_t n_shards, uint64_t shard_words,
                                  uint32_t my, uint64_t cap, hetm_log_entry* const* d_peer_out,
                                  unsigned long long* const* d_peer_counts, unsigned long long* d_totals,
                                  void* d_scratch, size_t scratch_bytes, const LaunchGeom& g, cudaStream_t s);

// Hand-written device primitives of the SCAN schedules (sort.cu).
// Stable LSD radix sort of (key, value) pairs on key bits [0, end_bit), n < 2^32.
size_t radix_sort_temp_bytes(uint64_t n, int end_bit);
cudaError_t radix_sort_init();  // once before any capture of radix_sort_pairs (kernel attributes)
cudaError_t radix_sort_pairs(const uint32_t* keys_in, uint32_t* keys_out, const uint32_t* vals_in, uint32_t* vals_out,
                             uint64_t n, int end_bit, void* temp, size_t temp_bytes, const LaunchGeom& g,
                             cudaStream_t s);
// out = the indices i < n with flags[i] != 0, in order; *d_count = their number.
size_t select_flagged_temp_bytes(uint64_t n);
cudaError_t select_flagged(const uint8_t* flags, uint64_t n, uint32_t* out, uint32_t* d_count, void* temp,
                           size_t temp_bytes, cudaStream_t s);
// Inclusive scan by key of {delta, last writer} over sorted traced-bank accesses
// (payload (4 i + k) << 1 | writer, delta indexed by 4 i + k): out[2j] = summed
// delta, out[2j+1] = last writing transaction (~0: none) since the key's start.
size_t seg_scan_temp_bytes(uint64_t n);
cudaError_t seg_scan_delta_writer(const uint32_t* keys, const uint32_t* pay, const unsigned long long* delta,
                                  uint64_t n, unsigned long long* out, void* temp, size_t temp_bytes, cudaStream_t s);

int query_geom(LaunchGeom* g, int device);

}  // namespace hetm_b200
