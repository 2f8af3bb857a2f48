// cache_sched.cu — the SCAN schedule of the cache batch (BASELINE configs[3]):
// abort-free execution of a GET/SET batch in input order (ticket = first + i).
//
// Every cache transaction touches exactly one set, so the serial execution in
// input order is, set by set, the subsequence of that set's transactions:
//   1. per transaction: sort key = its set (sentinel when the set lies outside
//      the shard), payload = input index; ticket = first + i;
//   2. radix sort of the (set, index) pairs on the set bits (sort.cu,
//      hand-written) — stable, so each set's transactions stay in input order;
//   3. one thread per set segment runs them in that order with the whole set
//      (64 words) in registers, storing the dirty words back at the segment's
//      end (it is the set's only accessor in this launch): hit / invalid /
//      LRU-victim choice, results,
//      LRU stamp = ticket + 1, write-set log slots, RS / WS / ChunkMap marks —
//      the same per-transaction rule as cache_tx.cu and the oracle's
//      cache_apply; at the segment's end the set lock word takes the version
//      lk_commit(ticket of the set's last update).
// No lock is taken and nothing retries: hot sets cost one thread a loop over
// their transactions instead of a chain of lock handoffs.
#include <algorithm>

#include "common.cuh"
#include "device_tm.cuh"
#include "kernels.h"

namespace hetm_b200 {

namespace {

constexpr unsigned kCsThreads = 128;
constexpr uint32_t kNoSet = 0xffffffffu;
constexpr int kWays = HETM_CACHE_WAYS;
constexpr int kWayWords = HETM_CACHE_WAY_WORDS;
constexpr int kSetWords = HETM_CACHE_SET_WORDS;
enum : int { kKey0 = 0, kKey1 = 1, kVal = 2, kLru = 6, kFlags = 7 };

unsigned grid_of(uint64_t n, unsigned threads, unsigned per_sm, int sms) {
    const uint64_t want = (n + threads - 1) / threads, cap = (uint64_t)per_sm * (uint64_t)sms;
    return (unsigned)std::max<uint64_t>(1, std::min(want, cap));
}
uint32_t bits_of(uint64_t x) {
    uint32_t b = 0;
    while (b < 64 && (1ull << b) < x) ++b;
    return b;
}

__global__ void cs_ticket_kernel(DevCounters* ctr, uint64_t n, unsigned long long* first) {
    *first = atomicAdd(&ctr->ticket, (unsigned long long)n);
}

__global__ void cs_keys_kernel(ShardView v, CacheGeom cg, const hetm_cache_tx* __restrict__ in, uint64_t n,
                               uint32_t* __restrict__ sets, uint32_t* __restrict__ pay,
                               unsigned long long* __restrict__ tickets, const unsigned long long* first,
                               DevCounters* ctr) {
    const unsigned long long t0 = *first, wbase = ld_relaxed(&ctr->wlog_base);
    unsigned oob = 0, any_set = 0;
    unsigned long long commits = 0;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t k0 = in[i].key[0], k1 = in[i].key[1];
        const uint64_t set = cache_set_of(k0, k1, cg.n_sets);
        const bool ok = cg.base_local + (set + 1) * kSetWords <= v.size_words;
        oob |= !ok;
        commits += ok;
        any_set |= ok && in[i].op != HETM_CACHE_GET;
        sets[i] = ok ? (uint32_t)set : kNoSet;
        pay[i] = (uint32_t)i;
        tickets[i] = ok ? t0 + i : ~0ull;
        if (!ok) {
            wlog_put(v, wbase, t0 + i, 0, ~0u);
            wlog_put(v, wbase, t0 + i, 1, ~0u);
        }
    }
    if (__any_sync(0xffffffffu, oob) && lane_id() == 0) atomicOr(&ctr->oob, 1u);
    // a SET writes up to 8 words: more than the write-set log's 2 slots
    if (__any_sync(0xffffffffu, any_set) && lane_id() == 0) ctr->wlog_overflow = 1;
    const unsigned long long c = warp_sum(commits);
    if (lane_id() == 0 && c) atomicAdd(&ctr->committed, c);
}

// Bitmap marks for the words of the set at s0 selected by mask: one probe (and
// at most one RED) per granule the set spans — 1 or 2 at the default 1 KiB.
__device__ __noinline__ void mark_mask(unsigned long long* bm, uint64_t s0, uint64_t mask, uint32_t shift) {
    if (!mask) return;
    const uint64_t g0 = s0 >> shift, g1 = (s0 + kSetWords - 1) >> shift;
    for (uint64_t g = g0; g <= g1; ++g) {
        const uint64_t lo = g << shift, hi = (g + 1) << shift;  // words of granule g
        const uint64_t a = lo > s0 ? lo - s0 : 0, b = hi - s0 < kSetWords ? hi - s0 : kSetWords;
        const uint64_t m = (b >= 64 ? ~0ull : (1ull << b) - 1) & ~((1ull << a) - 1);
        if ((mask & m) && !test_bit(bm, g)) set_bit(bm, g);
    }
}

// The transaction records in set-sorted order (one parallel gather), so a
// segment's records are contiguous: the serial walk of a hot set then reads
// lines already in L1/L2 instead of one random DRAM record per step.
__global__ void cs_gather_kernel(const hetm_cache_tx* __restrict__ in, uint64_t n, const uint32_t* __restrict__ pay,
                                 const uint32_t* __restrict__ sets, hetm_cache_tx* __restrict__ recs,
                                 uint8_t* __restrict__ start) {
    for (uint64_t j = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; j < n; j += (uint64_t)gridDim.x * blockDim.x) {
        recs[j] = in[pay[j]];
        const uint32_t set = sets[j];
        start[j] = set != kNoSet && (j == 0 || sets[j - 1] != set);  // a set segment begins here
    }
}

// One 256-bit load: the value words of two adjacent cells {v0, m0, v1, m1}.
__device__ __forceinline__ void ld_vals2(const Cell* c, uint64_t& v0, uint64_t& v1) {
    asm volatile("{\n\t.reg .b64 m0, m1;\n\tld.relaxed.gpu.global.v4.u64 {%0, m0, %1, m1}, [%2];\n\t}"
                 : "=l"(v0), "=l"(v1)
                 : "l"(c)
                 : "memory");
}

// One thread per set segment (the segment starts compacted first, so no lane
// idles on a non-start position).  The 32 tag words {key0, key1, lru, flags}
// of the 8 ways live in registers (predicated updates); the 32 value words in
// shared memory, column-major per thread (conflict-free), indexed by way —
// a runtime index into registers would spill, and selecting over all 32
// value registers per transaction cost most of the instructions.  The next
// record is loaded while the current one runs; dirty words are stored once,
// at the segment's end.

__global__ void __launch_bounds__(kCsThreads) cs_run_kernel(ShardView v, CacheGeom cg,
                                                            const hetm_cache_tx* __restrict__ recs, uint64_t n,
                                                            const uint32_t* __restrict__ sets,
                                                            const uint32_t* __restrict__ pay,
                                                            const uint32_t* __restrict__ starts,
                                                            const uint32_t* __restrict__ n_starts,
                                                            hetm_cache_result* __restrict__ res,
                                                            const unsigned long long* first, DevCounters* ctr) {
    __shared__ uint64_t sval[4 * kWays][kCsThreads];  // [way * 4 + q][thread]
    uint64_t* val = &sval[0][threadIdx.x];             // val[(way * 4 + q) * kCsThreads]
    const unsigned long long t0 = *first, wbase = ld_relaxed(&ctr->wlog_base);
    const uint64_t m = *n_starts;
    for (uint64_t k = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; k < m; k += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t j = starts[k];
        const uint32_t set = sets[j];
        const uint64_t s0 = cg.base_local + (uint64_t)set * kSetWords;
        Cell* cs = v.cells + s0;
        uint64_t k0[kWays], k1[kWays], lru[kWays], fl[kWays];
#pragma unroll
        for (int a = 0; a < kWays; ++a) {
            ld_vals2(&cs[a * kWayWords + kKey0], k0[a], k1[a]);
            ld_vals2(&cs[a * kWayWords + kLru], lru[a], fl[a]);
            uint64_t x0, x1, x2, x3;
            ld_vals2(&cs[a * kWayWords + kVal], x0, x1);
            ld_vals2(&cs[a * kWayWords + kVal + 2], x2, x3);
            val[(a * 4 + 0) * kCsThreads] = x0;
            val[(a * 4 + 1) * kCsThreads] = x1;
            val[(a * 4 + 2) * kCsThreads] = x2;
            val[(a * 4 + 3) * kCsThreads] = x3;
        }
        uint64_t rs_mask = 0, ws_mask = 0;  // words of the set read / written by the segment
        unsigned long long last_update = ~0ull;
        uint64_t i = pay[j];
        hetm_cache_tx r = recs[j];
        for (uint64_t jj = j;;) {
            const bool more = jj + 1 < n && sets[jj + 1] == set;  // load the next transaction ahead
            uint64_t i_next = 0;
            hetm_cache_tx r_next;
            if (more) {
                i_next = pay[jj + 1];
                r_next = recs[jj + 1];
            }
            const unsigned long long t = t0 + i;
            const bool is_get = r.op == HETM_CACHE_GET;
            int hit = kWays, invalid = kWays, lru_way = 0;
#pragma unroll
            for (int a = kWays - 1; a >= 0; --a) {  // lowest index wins every tie
                if ((fl[a] & 1) && k0[a] == r.key[0] && k1[a] == r.key[1]) hit = a;
                if (!(fl[a] & 1)) invalid = a;
            }
            uint64_t lru_min = lru[0];
#pragma unroll
            for (int a = 1; a < kWays; ++a)
                if (lru[a] < lru_min) {
                    lru_min = lru[a];
                    lru_way = a;
                }
            int target;
            uint32_t status;
            if (is_get) {
                target = hit;
                status = hit < kWays ? HETM_CACHE_HIT : HETM_CACHE_MISS;
            } else if (hit < kWays) {
                target = hit;
                status = HETM_CACHE_UPDATED;
            } else if (invalid < kWays) {
                target = invalid;
                status = HETM_CACHE_INSERTED;
            } else {
                target = lru_way;
                status = HETM_CACHE_EVICTED;
            }
            hetm_cache_result out;
            out.status = status;
            out.way = (uint32_t)target;
            if (target < kWays) {
                uint64_t* tv = val + (uint64_t)target * 4 * kCsThreads;
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    out.value[q] = is_get ? tv[q * kCsThreads] : r.value[q];
                    if (!is_get) tv[q * kCsThreads] = r.value[q];
                }
                const bool fill = !is_get && status != HETM_CACHE_UPDATED;
#pragma unroll
                for (int a = 0; a < kWays; ++a) {
                    const bool mt = a == target;
                    k0[a] = (mt && fill) ? r.key[0] : k0[a];
                    k1[a] = (mt && fill) ? r.key[1] : k1[a];
                    fl[a] = (mt && fill) ? 1ull : fl[a];
                    lru[a] = mt ? t + 1 : lru[a];
                }
                const uint32_t wl = (uint32_t)(target * kWayWords);
                rs_mask |= 0xfull << (wl + kVal);
                ws_mask |= (is_get ? (1ull << kLru)
                                   : (status == HETM_CACHE_UPDATED ? (0x1full << kVal) : 0xffull)) << wl;
                last_update = t;
                wlog_put(v, wbase, t, 0, is_get ? (uint32_t)(s0 + wl + kLru) : ~0u);  // the LRU touch
            } else {
#pragma unroll
                for (int q = 0; q < 4; ++q) out.value[q] = 0;
                wlog_put(v, wbase, t, 0, ~0u);
            }
            wlog_put(v, wbase, t, 1, ~0u);
            if (res) res[i] = out;
            if (!more) break;
            ++jj;
            i = i_next;
            r = r_next;
        }
        // every transaction read the tag words of all ways
#pragma unroll
        for (int a = 0; a < kWays; ++a)
            rs_mask |= ((1ull << kKey0) | (1ull << kKey1) | (1ull << kLru) | (1ull << kFlags)) << (a * kWayWords);
#pragma unroll
        for (int a = 0; a < kWays; ++a) {
            const uint64_t wm = ws_mask >> (a * kWayWords);
            if (!(wm & 0xffull)) continue;
            Cell* way = cs + a * kWayWords;
            if (wm & (1ull << kKey0)) way[kKey0].value = k0[a];
            if (wm & (1ull << kKey1)) way[kKey1].value = k1[a];
#pragma unroll
            for (int q = 0; q < 4; ++q)
                if (wm & (1ull << (kVal + q))) way[kVal + q].value = val[(a * 4 + q) * kCsThreads];
            if (wm & (1ull << kLru)) way[kLru].value = lru[a];
            if (wm & (1ull << kFlags)) way[kFlags].value = fl[a];
        }
        mark_mask(v.rs, s0, rs_mask, v.gran_shift);
        mark_mask(v.ws, s0, ws_mask, v.gran_shift);
        mark_mask(v.chunk, s0, ws_mask, v.chunk_shift);
        if (last_update != ~0ull) cs[0].meta = lk_commit(last_update);  // the set lock's version
    }
}

}  // namespace

size_t cache_sched_temp_bytes(uint64_t n, uint64_t n_sets) {
    const int end_bit = (int)std::min<uint32_t>(32, bits_of(n_sets) + 1);
    auto al = [](size_t x) { return (x + 255) & ~size_t(255); };
    // [sets in/out | payload in/out | starts | records | start flags | first | n_starts | sort / select temp]
    return 5 * al(n * 4) + al(n * sizeof(hetm_cache_tx)) + al(n) + 512 +
           al(std::max(radix_sort_temp_bytes(n, end_bit), select_flagged_temp_bytes(n)));
}

cudaError_t launch_cache_sched(const ShardView& v, const CacheGeom& cg, const hetm_cache_tx* d_in, uint64_t n,
                               unsigned long long* d_tickets, hetm_cache_result* d_res, DevCounters* ctr, void* temp,
                               size_t temp_bytes, const LaunchGeom& g, cudaStream_t s) {
    if (n == 0) return cudaSuccess;
    if (n >= (1ull << 32)) return cudaErrorInvalidValue;
    auto al = [](size_t x) { return (x + 255) & ~size_t(255); };
    char* p = static_cast<char*>(temp);
    uint32_t* sets = reinterpret_cast<uint32_t*>(p);
    uint32_t* sets_s = reinterpret_cast<uint32_t*>(p + al(n * 4));
    uint32_t* pay = reinterpret_cast<uint32_t*>(p + 2 * al(n * 4));
    uint32_t* pay_s = reinterpret_cast<uint32_t*>(p + 3 * al(n * 4));
    uint32_t* starts = reinterpret_cast<uint32_t*>(p + 4 * al(n * 4));
    auto* recs = reinterpret_cast<hetm_cache_tx*>(p + 5 * al(n * 4));
    auto* start = reinterpret_cast<uint8_t*>(p + 5 * al(n * 4) + al(n * sizeof(hetm_cache_tx)));
    const size_t off = 5 * al(n * 4) + al(n * sizeof(hetm_cache_tx)) + al(n);
    auto* first = reinterpret_cast<unsigned long long*>(p + off);
    auto* n_starts = reinterpret_cast<uint32_t*>(p + off + 256);
    void* sort_tmp = p + off + 512;
    const size_t sort_bytes = temp_bytes - (off + 512);
    const int end_bit = (int)std::min<uint32_t>(32, bits_of(cg.n_sets) + 1);
    cs_ticket_kernel<<<1, 1, 0, s>>>(ctr, n, first);
    cs_keys_kernel<<<grid_of(n, 256, 8, g.sm_count), 256, 0, s>>>(v, cg, d_in, n, sets, pay, d_tickets, first, ctr);
    cudaError_t e = radix_sort_pairs(sets, sets_s, pay, pay_s, n, end_bit, sort_tmp, sort_bytes, g, s);
    if (e != cudaSuccess) return e;
    cs_gather_kernel<<<grid_of(n, 256, 8, g.sm_count), 256, 0, s>>>(d_in, n, pay_s, sets_s, recs, start);
    e = select_flagged(start, n, starts, n_starts, sort_tmp, sort_bytes, s);
    if (e != cudaSuccess) return e;
    cs_run_kernel<<<grid_of(n, kCsThreads, 16, g.sm_count), kCsThreads, 0, s>>>(v, cg, recs, n, sets_s, pay_s, starts,
                                                                              n_starts, d_res, first, ctr);
    return cudaGetLastError();
}

}  // namespace hetm_b200
