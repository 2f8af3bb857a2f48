// common.cuh — HBM layout and sm_100a memory-model helpers for the HeTM kernels.
//
// Device replica layout: one 16-byte WORD CELL per STMR word,
//     { value, meta }                       (two cells per 32-B sector)
// so every per-word operation of the hot path touches exactly one sector:
//   * the batch TM reads {value, meta} with one 128-bit single-copy-atomic
//     load and commits {new value, unlocked new version} with one 128-bit
//     store (no separate lock table, no fence between write-back and release);
//   * validation raises the TsArray entry held in `meta`
//     and stores the winning value in the same sector.
// `meta` is the batch TM's versioned lock word between validation phases and
// the word's TS after a host write was applied to it (device_tm.cuh):
//     FINAL(63) | 0 | owner(61..32) | version(31..0)    lock / version word
//     0 | TS-tag(62) | host ts(61..0)                    TS word (unlocked)
// The two never coexist in time: validation/apply never overlaps a batch,
// and a batch treats a TS word as an unlocked word of one reserved version.
// The raw-op / merge boundary still sees a plain array of 64-bit words
// (SPEC.md:78): gather/scatter kernels convert at the edge, and devShadow is a
// plain word array so dirty chunks DMA straight to the host replica.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "hetm_b200/capi.h"

namespace hetm_b200 {

struct alignas(16) Cell {
    uint64_t value;           // the STMR word (devReplica)
    unsigned long long meta;  // versioned lock word, or TS-tag | ts
};
static_assert(sizeof(Cell) == 16, "two cells per 32-B sector");

constexpr unsigned long long kTsTag = 1ull << 62;
// meta of a word whose freshest applied host write has timestamp ts
__host__ __device__ __forceinline__ unsigned long long ts_meta(uint64_t ts) { return kTsTag | ts; }

// Minimum capacity of the apply kernel's restore queue (entries); the handle
// grows it to a quarter of the largest apply launch (kernels.h RestoreQueue).
constexpr uint64_t kRestoreCap = 1ull << 20;

// Device-wide counters, one per handle (HBM, 128-B aligned).
struct DevCounters {
    unsigned long long ticket;      // next commit ticket (global serial order)
    unsigned long long committed;   // last batch
    unsigned long long aborts;      // last batch: aborted attempts
    unsigned long long livelocked;  // last batch
    unsigned long long retried;     // last batch: transactions committed after >= 2 aborted attempts
    unsigned long long round_max_ts;// max log ts seen this round
    unsigned int conflict;          // round conflictFlag
    unsigned int nonmonotone;       // a log ts <= ts_floor was seen
    unsigned int oob;               // an address outside this shard was seen
    unsigned int pad0;
    unsigned long long restore_n;    // apply: raced entries queued for restore_kernel
    unsigned long long restore_done; // restore_kernel: finished blocks
    unsigned long long ts_floor;     // max log ts of all previous rounds (device-maintained)
    unsigned long long wlog_base;    // first commit ticket of the round (write-set log origin)
    unsigned long long wlog_overflow;// a committed write set did not fit the write-set log
    unsigned long long apply_dups;   // apply: exchange put-backs so far (monotone; the host judges deltas)
    unsigned long long pad[18];      // diagnostics (phase clocks / ticket counts)
};

static_assert(sizeof(DevCounters) == 256, "two 128-B lines");

// Kernel-wide view of one device's STMR shard and its metadata.
struct ShardView {
    Cell* cells;               // devReplica + locks + TS (size_words cells)
    uint64_t base;             // global index of cells[0]
    uint64_t size_words;
    unsigned long long* rs;    // RS bitmap words
    unsigned long long* ws;    // WS bitmap words
    unsigned long long* chunk; // ChunkMap words
    uint32_t gran_shift;       // bit = local_word >> gran_shift   (gran = 8 << gran_shift)
    uint32_t chunk_shift;      // chunk = local_word >> chunk_shift
    uint32_t* wlog;            // device write-set log (nullptr: disabled, shard >= 2^32 words)
    uint64_t wlog_slots;       // its capacity in slots
    unsigned long long* wlog_ovf; // set when a committed write set did not fit (DevCounters::wlog_overflow)
    uint32_t serial;           // deterministic single-worker mode (HETM_CFG_DETERMINISTIC)
    unsigned long long* trace; // checker trace of the batch (nullptr: off): HETM_TRACE_TX_WORDS per tx index
    unsigned int* stripes;     // bank kernel lock-stripe table (phased_tx.cuh KO_STRIPES; nullptr: cell locks)
    uint32_t stripe_shift;       // stripe = (loc * 2^64/phi) >> stripe_shift  (64 - log2 stripes)
};

// Checker trace record of one committed batch transaction (capi.h
// hetm_dev_trace_next_batch): [0] ticket, [1..4] values of the read words in
// program order, [5..6] values read by the read-modify-writes, [7..8] values
// written, [9..11] reserved.  Transactions that did not commit keep ~0 in [0].
constexpr int kTraceWords = 12;

// First transaction and stride of the calling thread in a batch kernel.  In the
// deterministic single-worker mode global thread 0 runs every
// transaction in input order, so ticket i = first ticket + i.
__device__ __forceinline__ void tx_range(const ShardView& v, uint64_t n, uint64_t& i, uint64_t& stride) {
    const uint64_t tid = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (v.serial) {
        i = tid == 0 ? 0 : n;
        stride = 1;
    } else {
        i = tid;
        stride = (uint64_t)gridDim.x * blockDim.x;
    }
}

// Cache region of HETM_KERNEL_CACHE (capi.h hetm_cache_*): n_sets sets of
// HETM_CACHE_SET_WORDS words from local word base_local.
struct CacheGeom {
    uint64_t base_local;
    uint64_t n_sets;  // power of two >= 2
};

// Key hash (splitmix64 finalizer over the two key words) and last-bit routing
// (PAPER.md:489): part = key0 & 1 owns the half [part*n/2, (part+1)*n/2).
__host__ __device__ __forceinline__ uint64_t cache_hash(uint64_t k0, uint64_t k1) {
    uint64_t z = k0 ^ (k1 * 0x9e3779b97f4a7c15ull);
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
    return z ^ (z >> 31);
}
__host__ __device__ __forceinline__ uint64_t cache_set_of(uint64_t k0, uint64_t k1, uint64_t n_sets) {
    const uint64_t half = n_sets >> 1;
    return (k0 & 1ull) * half + (cache_hash(k0, k1) & (half - 1));
}

// Device write-set log: slot 2*(ticket - round's first ticket) + j holds the
// local index of the j-th written word of the committed transaction (~0u:
// none).  Consecutive tickets of a warp store contiguously; the merge turns
// the log into a compact {word, value} delta.
__device__ __forceinline__ void wlog_put(const ShardView& v, unsigned long long wbase, unsigned long long t, int j,
                                         uint32_t loc) {
    const unsigned long long s = (t - wbase) * 2ull + (unsigned)j;
    if (s < v.wlog_slots) v.wlog[s] = loc;
    else if (v.wlog) *v.wlog_ovf = 1;  // the merge and rollback fall back to dirty chunks
}

__device__ __forceinline__ uint64_t ld_relaxed(const uint64_t* p) {
    uint64_t v;
    asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ unsigned long long ld_relaxed(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ unsigned int ld_relaxed(const unsigned int* p) {
    unsigned int v;
    asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_relaxed(unsigned int* p, unsigned int v) {
    asm volatile("st.relaxed.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void st_relaxed(uint64_t* p, uint64_t v) {
    asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ void st_relaxed(unsigned long long* p, unsigned long long v) {
    asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

// {value, lock} of a cell as ONE single-copy-atomic 128-bit access
// (LDG.E.128.STRONG.GPU / STG.E.128.STRONG.GPU; the same instructions
// libcu++ uses for 16-byte cuda::atomic).
__device__ __forceinline__ void ld_pair(const Cell* c, uint64_t& value, unsigned long long& lock) {
    asm volatile("{\n\t.reg .b128 t;\n\tld.relaxed.gpu.global.b128 t, [%2];\n\tmov.b128 {%0, %1}, t;\n\t}"
                 : "=l"(value), "=l"(lock)
                 : "l"(c)
                 : "memory");
}
__device__ __forceinline__ void st_pair(Cell* c, uint64_t value, unsigned long long lock) {
    asm volatile("{\n\t.reg .b128 t;\n\tmov.b128 t, {%1, %2};\n\tst.relaxed.gpu.global.b128 [%0], t;\n\t}" ::"l"(c),
                 "l"(value), "l"(lock)
                 : "memory");
}

__device__ __forceinline__ void set_bit(unsigned long long* words, uint64_t bit) {
    atomicOr(&words[bit >> 6], 1ull << (bit & 63));  // REDG.E.OR.64 (result unused)
}
__device__ __forceinline__ void red_or_bit(unsigned long long* words, uint64_t bit) {
    asm volatile("red.relaxed.gpu.global.or.b64 [%0], %1;" ::"l"(&words[bit >> 6]), "l"(1ull << (bit & 63)) : "memory");
}
__device__ __forceinline__ bool test_bit(const unsigned long long* words, uint64_t bit) {
    return (words[bit >> 6] >> (bit & 63)) & 1ull;
}

__device__ __forceinline__ unsigned lane_id() { return threadIdx.x & 31u; }

// Warp-collective (all 32 lanes): set bit `bit` of `words` where `pred`, for
// lanes whose bits arrive in NONDECREASING word order across the warp (a
// sorted stream): each contiguous run of lanes naming the same word ORs its
// masks together and its first lane issues one probe-gated atomic.  Lanes with
// pred false split runs but stay correct.
__device__ __forceinline__ void warp_set_bits_sorted(unsigned long long* words, uint64_t bit, bool pred) {
    const unsigned lane = lane_id();
    const uint64_t w = pred ? bit >> 6 : ~0ull;
    unsigned long long m = pred ? 1ull << (bit & 63) : 0ull;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {  // suffix OR within the run
        const uint64_t wd = __shfl_down_sync(0xffffffffu, w, d);
        const unsigned long long md = __shfl_down_sync(0xffffffffu, m, d);
        if (lane + d < 32 && wd == w) m |= md;
    }
    const uint64_t wprev = __shfl_up_sync(0xffffffffu, w, 1);
    if (pred && (lane == 0 || wprev != w) && (words[w] & m) != m) atomicOr(&words[w], m);
}


template <typename T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

}  // namespace hetm_b200
