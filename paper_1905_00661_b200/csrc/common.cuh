// common.cuh — sm_100a memory-model helpers shared by the HeTM device kernels.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "hetm_b200/capi.h"

namespace hetm_b200 {

// Device-wide counters, one per handle (HBM, 128-B aligned).
struct DevCounters {
    unsigned long long ticket;      // next commit ticket (global serial order)
    unsigned long long committed;   // last batch
    unsigned long long aborts;      // last batch: aborted attempts
    unsigned long long livelocked;  // last batch
    unsigned long long round_max_ts;// max log ts seen this round
    unsigned int conflict;          // round conflictFlag
    unsigned int nonmonotone;       // a log ts <= ts_floor was seen
    unsigned int oob;               // an address outside this shard was seen
    unsigned int pad0;
    unsigned long long pad[9];
};

// Kernel-wide view of one device's STMR shard and its metadata.
struct ShardView {
    uint64_t* stmr;            // devReplica (size_words)
    uint64_t base;             // global index of stmr[0]
    uint64_t size_words;
    unsigned long long* rs;    // RS bitmap words
    unsigned long long* ws;    // WS bitmap words
    unsigned long long* chunk; // ChunkMap words
    uint32_t gran_shift;       // bit = local_word >> gran_shift   (gran = 8 << gran_shift)
    uint32_t chunk_shift;      // chunk = local_word >> chunk_shift
};

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
__device__ __forceinline__ void st_relaxed(uint64_t* p, uint64_t v) {
    asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ void st_relaxed(unsigned long long* p, unsigned long long v) {
    asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ void st_release(unsigned long long* p, unsigned long long v) {
    asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ void fence_acq_rel() { asm volatile("fence.acq_rel.gpu;" ::: "memory"); }

// Streaming (read-once) 128-bit load that does not allocate in L1.
__device__ __forceinline__ uint4 ld_stream_v4(const void* p) {
    uint4 r;
    asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
                 : "l"(p));
    return r;
}

__device__ __forceinline__ void set_bit(unsigned long long* words, uint64_t bit) {
    atomicOr(&words[bit >> 6], 1ull << (bit & 63));  // REDG.E.OR.64 (result unused)
}
__device__ __forceinline__ bool test_bit(const unsigned long long* words, uint64_t bit) {
    return (words[bit >> 6] >> (bit & 63)) & 1ull;
}

__device__ __forceinline__ unsigned lane_id() { return threadIdx.x & 31u; }

template <typename T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

}  // namespace hetm_b200
