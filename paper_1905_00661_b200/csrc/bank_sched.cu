// bank_sched.cu — the SCAN schedule of the bank batch: a skew-proof,
// abort-free execution of a whole batch in input order (ticket = first + i).
//
// A bank transaction's writes are read-modify-writes with known deltas
// (acct0 -= amount, acct1 += amount; acct2/acct3 only read), so the serial
// execution of the batch in input order is a segmented prefix sum:
//   1. keys: one 64-bit key per access, loc << sh | i << 2 | k (sh = bits of
//      4n), so sorting groups each account's accesses in input order;
//   2. CUB radix sort of the 4n keys;
//   3. CUB inclusive scan-by-account of {delta, last writer}: the delta of an
//      access is the transaction's net effect on that account (last write wins
//      when acct0 == acct1), carried by the first slot naming the account;
//   4. one pass over the sorted accesses: at the end of each account's segment
//      the final value and version (lk_commit of the last writer's ticket) are
//      stored and the WS / chunk bits set, at its start the RS bit; every
//      access of slot 0/1 writes its ticket and write-set log slot.  With a
//      trace armed, a read-only pass first records each access's pre-value.
// Cost is independent of skew (no locks, no retries): at zipf 0.99 the
// optimistic PR-STM kernel serializes ~10^5 commits on the hottest account.
// The result is exactly the deterministic single-worker mode.
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>
#include <thrust/iterator/transform_iterator.h>

#include "common.cuh"
#include "device_tm.cuh"
#include "kernels.h"

#include <algorithm>

namespace hetm_b200 {

namespace {

constexpr unsigned kSchedThreads = 256;
constexpr unsigned long long kNone = ~0ull;

struct DeltaW {  // scan value: summed delta, last writing transaction (input index) or kNone
    unsigned long long d, w;
};
struct DeltaWOp {
    __host__ __device__ DeltaW operator()(const DeltaW& a, const DeltaW& b) const {
        return DeltaW{a.d + b.d, b.w != kNone ? b.w : a.w};
    }
};

struct LocOf {  // segment key: the account (sentinels form their own segment)
    using result_type = unsigned long long;
    uint32_t sh;
    __host__ __device__ unsigned long long operator()(unsigned long long key) const { return key >> sh; }
};

__device__ __forceinline__ void load_accts(const hetm_bank_tx* in, uint64_t i, uint64_t base, uint64_t (&a)[4],
                                           uint64_t& amount) {
    const uint64_t* rec = reinterpret_cast<const uint64_t*>(in + i);
    const uint64_t w01 = __ldg(rec), w23 = __ldg(rec + 1);
    amount = __ldg(rec + 2);
    a[0] = (w01 & 0xffffffffu) - base;
    a[1] = (w01 >> 32) - base;
    a[2] = (w23 & 0xffffffffu) - base;
    a[3] = (w23 >> 32) - base;
}

struct DeltaOf {  // the access's scan value
    using result_type = DeltaW;
    const hetm_bank_tx* in;
    uint64_t base;
    uint32_t sh;
    __device__ DeltaW operator()(unsigned long long key) const {
        if (key == kNone) return DeltaW{0, kNone};
        const uint64_t i = (key & ((1ull << sh) - 1)) >> 2;
        const int k = (int)(key & 3);
        uint64_t a[4], amount;
        load_accts(in, i, base, a, amount);
        for (int q = 0; q < k; ++q)
            if (a[q] == a[k]) return DeltaW{0, kNone};  // not the first slot naming this account
        if (a[k] == a[1]) return DeltaW{amount, i};   // the last write wins (acct1 after acct0)
        if (a[k] == a[0]) return DeltaW{0ull - amount, i};
        return DeltaW{0, kNone};
    }
};

__global__ void sched_keys_kernel(ShardView v, const hetm_bank_tx* __restrict__ in, uint64_t n, uint32_t sh,
                                  unsigned long long* __restrict__ keys, unsigned long long* __restrict__ tickets,
                                  const unsigned long long* first, DevCounters* ctr) {
    const uint64_t base = v.base, size_words = v.size_words;
    const unsigned long long t0 = *first, wbase = ld_relaxed(&ctr->wlog_base);
    unsigned oob = 0;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
        uint64_t a[4], amount;
        load_accts(in, i, base, a, amount);
        const bool ok = a[0] < size_words && a[1] < size_words && a[2] < size_words && a[3] < size_words;
        oob |= !ok;
        if (!ok) {  // rejected (outside this shard): no ticket, its log slots empty
            tickets[i] = kNone;
            wlog_put(v, wbase, t0 + i, 0, ~0u);
            wlog_put(v, wbase, t0 + i, 1, ~0u);
        }
#pragma unroll
        for (int k = 0; k < 4; ++k) keys[4 * i + k] = ok ? (a[k] << sh | i << 2 | (uint64_t)k) : kNone;
    }
    if (__any_sync(0xffffffffu, oob) && lane_id() == 0) atomicOr(&ctr->oob, 1u);
}

// First ticket of the batch; tickets of rejected (out-of-shard) transactions
// stay unused, their write-set log slots empty.
__global__ void sched_ticket_kernel(DevCounters* ctr, uint64_t n, unsigned long long* first) {
    *first = atomicAdd(&ctr->ticket, (unsigned long long)n);
}

// Read-only pass (traced batches): the value every access reads = the account's
// batch-start value + the deltas of the earlier transactions.
__global__ void sched_trace_kernel(ShardView v, const hetm_bank_tx* __restrict__ in, uint64_t n4, uint32_t sh,
                                   const unsigned long long* __restrict__ keys, const DeltaW* __restrict__ incl,
                                   const unsigned long long* first) {
    const unsigned long long t0 = *first;
    const DeltaOf dof{in, v.base, sh};
    for (uint64_t j = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; j < n4; j += (uint64_t)gridDim.x * blockDim.x) {
        const unsigned long long key = keys[j];
        if (key == kNone) continue;
        const uint64_t loc = key >> sh, i = (key & ((1ull << sh) - 1)) >> 2;
        const int k = (int)(key & 3);
        // pre-value: exclusive of this transaction's own delta, which sits on its
        // first slot naming the account (the entry itself or an earlier one of i)
        uint64_t jj = j;
        while (jj > 0 && (keys[jj - 1] >> 2) == (key >> 2)) --jj;  // first entry of (loc, i)
        const unsigned long long pre = v.cells[loc].value + incl[jj].d - dof(keys[jj]).d;
        unsigned long long* r = v.trace + i * kTraceWords;
        if (k == 0) r[0] = t0 + i;
        r[1 + k] = pre;
        if (k < 2) {
            uint64_t a[4], amount;
            load_accts(in, i, v.base, a, amount);
            r[5 + k] = pre;
            r[7 + k] = k == 0 ? pre - amount : pre + amount;
        }
    }
}

__global__ void sched_commit_kernel(ShardView v, uint64_t n4, uint32_t sh, const unsigned long long* __restrict__ keys,
                                    const DeltaW* __restrict__ incl, const unsigned long long* first,
                                    unsigned long long* __restrict__ tickets, DevCounters* ctr) {
    const unsigned long long t0 = *first;
    const unsigned long long wbase = ld_relaxed(&ctr->wlog_base);
    unsigned long long commits = 0;
    for (uint64_t j = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; j < n4; j += (uint64_t)gridDim.x * blockDim.x) {
        const unsigned long long key = keys[j];
        if (key == kNone) continue;
        const uint64_t loc = key >> sh, i = (key & ((1ull << sh) - 1)) >> 2;
        const int k = (int)(key & 3);
        const unsigned long long t = t0 + i;
        if (k == 0) {
            tickets[i] = t;
            ++commits;
        }
        if (k < 2) wlog_put(v, wbase, t, k, (uint32_t)loc);
        const bool seg_first = j == 0 || (keys[j - 1] >> sh) != loc;
        const bool seg_last = j + 1 == n4 || (keys[j + 1] >> sh) != loc;
        if (seg_first) set_bit(v.rs, loc >> v.gran_shift);  // every access reads (RS = reads U writes)
        if (seg_last && incl[j].w != kNone) {
            const Cell c{v.cells[loc].value + incl[j].d, lk_commit(t0 + incl[j].w)};
            st_pair(&v.cells[loc], c.value, c.meta);
            set_bit(v.ws, loc >> v.gran_shift);
            set_bit(v.chunk, loc >> v.chunk_shift);
        }
    }
    const unsigned long long c = warp_sum(commits);
    if (lane_id() == 0 && c) atomicAdd(&ctr->committed, c);
}

unsigned grid_for(uint64_t n, unsigned threads, unsigned blocks_per_sm, int sms) {
    const uint64_t want = (n + threads - 1) / threads, cap = (uint64_t)blocks_per_sm * (uint64_t)sms;
    return (unsigned)std::max<uint64_t>(1, std::min(want, cap));
}

uint32_t bits_for(uint64_t x) {  // bits to hold values < x
    uint32_t b = 0;
    while (b < 64 && (1ull << b) < x) ++b;
    return b;
}

}  // namespace

// Hot-spot estimate of a device-resident bank batch (AUTO on the device-
// pointer path): one CTA inserts the accounts of kEstTx sampled transactions
// into a shared-memory hash table of {account, count} and stores the largest
// count to *out (mapped host memory: the next batch reads it without a sync).
constexpr unsigned kEstThreads = 1024, kEstTx = 2048, kEstSlots = 1u << 14;  // 8 K keys, load 0.5
constexpr size_t kEstSmem = kEstSlots * sizeof(unsigned long long);           // 128 KiB

__global__ void __launch_bounds__(kEstThreads) hot_estimate_kernel(const hetm_bank_tx* __restrict__ in, uint64_t n,
                                                                   uint32_t* out) {
    extern __shared__ unsigned long long slot[];  // account << 32 | count; ~0 = empty
    for (unsigned q = threadIdx.x; q < kEstSlots; q += blockDim.x) slot[q] = ~0ull;
    __syncthreads();
    const uint64_t S = n < kEstTx ? n : kEstTx, stride = n / S;
    unsigned best = 0;
    for (uint64_t q = threadIdx.x; q < 4 * S; q += blockDim.x) {
        const uint32_t a = in[(q >> 2) * stride].acct[q & 3];
        uint32_t h = (uint32_t)((a * 0x9e3779b97f4a7c15ull) >> 50);  // 14 bits
        for (;;) {
            unsigned long long cur = slot[h];
            if (cur == ~0ull) {
                cur = atomicCAS(&slot[h], ~0ull, (unsigned long long)a << 32 | 1u);
                if (cur == ~0ull) {
                    best = best > 1u ? best : 1u;
                    break;
                }
            }
            if ((uint32_t)(cur >> 32) == a) {
                const unsigned c = (unsigned)(atomicAdd(&slot[h], 1ull) & 0xffffffffu) + 1u;
                best = best > c ? best : c;
                break;
            }
            h = (h + 1) & (kEstSlots - 1);
        }
    }
    __shared__ unsigned block_best;
    if (threadIdx.x == 0) block_best = 0;
    __syncthreads();
    atomicMax(&block_best, best);
    __syncthreads();
    if (threadIdx.x == 0) *reinterpret_cast<volatile uint32_t*>(out) = block_best;
}

cudaError_t launch_bank_hot_estimate(const hetm_bank_tx* d_in, uint64_t n, uint32_t* out, cudaStream_t s) {
    if (n == 0) return cudaSuccess;
    static const cudaError_t attr =
        cudaFuncSetAttribute(hot_estimate_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kEstSmem);
    if (attr != cudaSuccess) return attr;
    hot_estimate_kernel<<<1, kEstThreads, kEstSmem, s>>>(d_in, n, out);
    return cudaGetLastError();
}

uint64_t bank_hot_estimate_sample(uint64_t n) { return n < kEstTx ? n : kEstTx; }

size_t bank_sched_temp_bytes(uint64_t n, uint64_t size_words) {
    const uint64_t n4 = 4 * n;
    const uint32_t sh = bits_for(n4), end_bit = std::min<uint32_t>(64, sh + bits_for(size_words) + 1);
    size_t a = 0, b = 0;
    cub::DeviceRadixSort::SortKeys(nullptr, a, (const unsigned long long*)nullptr, (unsigned long long*)nullptr,
                                   (int64_t)n4, 0, (int)end_bit);
    auto ki = thrust::make_transform_iterator((const unsigned long long*)nullptr, LocOf{sh});
    auto vi = thrust::make_transform_iterator((const unsigned long long*)nullptr, DeltaOf{nullptr, 0, sh});
    cub::DeviceScan::InclusiveScanByKey(nullptr, b, ki, vi, (DeltaW*)nullptr, DeltaWOp{}, (int64_t)n4);
    auto al = [](size_t x) { return (x + 255) & ~size_t(255); };
    // [keys | sorted keys | scan | first ticket | cub temp]
    return al(n4 * 8) * 2 + al(n4 * sizeof(DeltaW)) + 256 + al(std::max(a, b));
}

cudaError_t launch_bank_sched(const ShardView& v, const hetm_bank_tx* d_in, uint64_t n, unsigned long long* d_tickets,
                              DevCounters* ctr, void* temp, size_t temp_bytes, const LaunchGeom& g, cudaStream_t s) {
    if (n == 0) return cudaSuccess;
    const uint64_t n4 = 4 * n;
    const uint32_t sh = bits_for(n4), end_bit = std::min<uint32_t>(64, sh + bits_for(v.size_words) + 1);
    auto al = [](size_t x) { return (x + 255) & ~size_t(255); };
    char* p = static_cast<char*>(temp);
    auto* keys = reinterpret_cast<unsigned long long*>(p);
    auto* sorted = reinterpret_cast<unsigned long long*>(p + al(n4 * 8));
    auto* incl = reinterpret_cast<DeltaW*>(p + 2 * al(n4 * 8));
    auto* first = reinterpret_cast<unsigned long long*>(p + 2 * al(n4 * 8) + al(n4 * sizeof(DeltaW)));
    void* cub_tmp = p + 2 * al(n4 * 8) + al(n4 * sizeof(DeltaW)) + 256;
    size_t cub_bytes = temp_bytes - (2 * al(n4 * 8) + al(n4 * sizeof(DeltaW)) + 256);
    const unsigned grid_tx = grid_for(n, kSchedThreads, 8, g.sm_count);
    const unsigned grid_acc = grid_for(n4, kSchedThreads, 8, g.sm_count);
    sched_ticket_kernel<<<1, 1, 0, s>>>(ctr, n, first);
    sched_keys_kernel<<<grid_tx, kSchedThreads, 0, s>>>(v, d_in, n, sh, keys, d_tickets, first, ctr);
    cudaError_t e = cub::DeviceRadixSort::SortKeys(cub_tmp, cub_bytes, keys, sorted, (int64_t)n4, 0, (int)end_bit, s);
    if (e != cudaSuccess) return e;
    auto ki = thrust::make_transform_iterator((const unsigned long long*)sorted, LocOf{sh});
    auto vi = thrust::make_transform_iterator((const unsigned long long*)sorted, DeltaOf{d_in, v.base, sh});
    e = cub::DeviceScan::InclusiveScanByKey(cub_tmp, cub_bytes, ki, vi, incl, DeltaWOp{}, (int64_t)n4,
                                             cub::Equality(), s);
    if (e != cudaSuccess) return e;
    if (v.trace) sched_trace_kernel<<<grid_acc, kSchedThreads, 0, s>>>(v, d_in, n4, sh, sorted, incl, first);
    sched_commit_kernel<<<grid_acc, kSchedThreads, 0, s>>>(v, n4, sh, sorted, incl, first, d_tickets, ctr);
    return cudaGetLastError();
}

}  // namespace hetm_b200
