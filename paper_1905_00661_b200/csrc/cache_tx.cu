// cache_tx.cu — MemcachedGPU-style GET/SET transactions on a set-associative
// cache held in the STMR (BASELINE configs[3]; SPEC.md:
// 585-608).  Layout and semantics: include/hetm_b200/capi.h (hetm_cache_*).
//
// Every transaction touches exactly one set, so the set is the lock granule:
// the versioned lock word of the set's first word cell guards all 64 words
// of the set (a striped lock table, as TL2/TinySTM hash many words to one
// lock).  One thread runs one transaction:
//   P1  acquire-load the set lock (must be free), then the 32 tag words
//       {key0, key1, lru, flags} of the 8 ways and the value words of the
//       target way (hit, or victim for a SET miss)
//   P2  update: CAS lock version -> FINAL|prio; read-only GET miss: none
//   P3  commit ticket (after the lock is held; before validation)
//   P4  read-only: fence, the set lock must still show the P1 version
//   P5  update: store the written words, then release the lock with version
//       ticket+1 (st.release orders the word stores before it)
// Serial order = ticket order (same argument as device_tm.cuh: the ticket is
// taken while the whole read set is protected).  An attempt blocked by a
// FINAL holder waits for that lock word to change and retries.
#include "common.cuh"
#include "device_tm.cuh"
#include "kernels.h"

namespace hetm_b200 {

constexpr int kCacheThreads = 128;
constexpr int kWays = HETM_CACHE_WAYS;
constexpr int kWayWords = HETM_CACHE_WAY_WORDS;
constexpr int kSetWords = HETM_CACHE_SET_WORDS;
enum : int { kKey0 = 0, kKey1 = 1, kVal = 2, kLru = 6, kFlags = 7 };
static_assert(kWays * kWayWords == kSetWords, "set layout");

__device__ __forceinline__ unsigned long long ld_acquire(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
// Two adjacent word cells {value, meta, value, meta} in one 256-bit access
// (LDG.E.ENL2.256.STRONG.GPU on sm_100a).
__device__ __forceinline__ void ld_cells2(const Cell* c, uint64_t& v0, uint64_t& v1) {
    asm volatile("{\n\t.reg .b64 m0, m1;\n\tld.relaxed.gpu.global.v4.u64 {%0, m0, %1, m1}, [%2];\n\t}"
                 : "=l"(v0), "=l"(v1)
                 : "l"(c)
                 : "memory");
}

__device__ __forceinline__ void st_release(unsigned long long* p, unsigned long long v) {
    asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

// RS/WS/ChunkMap marks for a run of words; consecutive words of one granule
// cost one RED (a whole 512-B set is one bit at the default 1 KiB).
__device__ __forceinline__ void mark_word(unsigned long long* bm, uint64_t loc, uint32_t shift, uint64_t& last) {
    const uint64_t b = loc >> shift;
    if (b != last) {
        set_bit(bm, b);
        last = b;
    }
}

__global__ void __launch_bounds__(kCacheThreads) cache_batch_kernel(ShardView v, CacheGeom cg,
                                                                    const hetm_cache_tx* __restrict__ in, uint64_t n,
                                                                    unsigned long long* __restrict__ tickets,
                                                                    hetm_cache_result* __restrict__ res,
                                                                    DevCounters* ctr, uint32_t max_attempts) {
    unsigned long long commits = 0, aborts = 0, livelocks = 0;
    unsigned oob = 0, wlog_full = 0;
    const unsigned long long wbase = ld_relaxed(&ctr->wlog_base);
    unsigned long long rng = 0x9e3779b97f4a7c15ull * ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x + 1);
    uint64_t i0, stride;
    tx_range(v, n, i0, stride);
    for (uint64_t i = i0; i < n; i += stride) {
        const hetm_cache_tx r = in[i];
        const uint64_t s0 = cg.base_local + cache_set_of(r.key[0], r.key[1], cg.n_sets) * kSetWords;
        if (s0 + kSetWords > v.size_words) {
            tickets[i] = ~0ull;
            oob = 1;
            continue;
        }
        Cell* set = v.cells + s0;
        unsigned long long* lockp = &set[0].meta;
        const bool is_get = r.op == HETM_CACHE_GET;
        for (uint32_t attempt = 1;; ++attempt) {
            // ---- P1
            const unsigned long long L = ld_acquire(lockp);
            bool ok = !(L & kLockFinal);
            unsigned long long block = ok ? 0ull : L;
            uint64_t k0[kWays], k1[kWays], lru[kWays], fl[kWays];
#pragma unroll
            for (int w = 0; w < kWays; ++w) {  // {key0, key1} and {lru, flags}: two 256-bit loads per way
                ld_cells2(&set[w * kWayWords + kKey0], k0[w], k1[w]);
                ld_cells2(&set[w * kWayWords + kLru], lru[w], fl[w]);
            }
            int hit = kWays, invalid = kWays, lru_way = 0;
#pragma unroll
            for (int w = kWays - 1; w >= 0; --w) {  // lowest index wins every tie
                if ((fl[w] & 1) && k0[w] == r.key[0] && k1[w] == r.key[1]) hit = w;
                if (!(fl[w] & 1)) invalid = w;
            }
#pragma unroll
            for (int w = 1; w < kWays; ++w)
                if (lru[w] < lru[lru_way]) lru_way = w;
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
            uint64_t val[4] = {0, 0, 0, 0};
            if (target < kWays) {
                ld_cells2(&set[target * kWayWords + kVal], val[0], val[1]);
                ld_cells2(&set[target * kWayWords + kVal + 2], val[2], val[3]);
            }
            // ---- P2 .. P5
            unsigned long long t = ~0ull;
            if (ok && target < kWays) {  // update transaction
                const unsigned long long prev = atomicCAS(lockp, L, kLockFinal | lk_make((uint32_t)(i + 1), lk_ver(L)));
                ok = prev == L;
                if (!ok && (prev & kLockFinal)) block = prev;
                if (ok) {
                    t = take_ticket(&ctr->ticket);
                    Cell* way = set + target * kWayWords;
                    if (!is_get) {
                        if (status != HETM_CACHE_UPDATED) {
                            st_relaxed(&way[kKey0].value, r.key[0]);
                            st_relaxed(&way[kKey1].value, r.key[1]);
                            st_relaxed(&way[kFlags].value, 1ull);
                        }
#pragma unroll
                        for (int q = 0; q < 4; ++q) st_relaxed(&way[kVal + q].value, r.value[q]);
                    }
                    st_relaxed(&way[kLru].value, t + 1);
                    st_release(lockp, lk_commit(t));
                }
            } else if (ok) {  // read-only GET miss: ticket, then validate the set lock
                t = take_ticket(&ctr->ticket);
                __threadfence();
                ok = ld_relaxed(lockp) == L;
            }
            if (ok) {
                tickets[i] = t;
                hetm_cache_result out;
#pragma unroll
                for (int q = 0; q < 4; ++q) out.value[q] = is_get ? val[q] : r.value[q];
                out.status = status;
                out.way = (uint32_t)target;
                if (res) res[i] = out;
                // bitmaps: tag words of every way (+ the target
                // way's values) read; written words -> WS and ChunkMap
                uint64_t last = ~0ull;
#pragma unroll
                for (int w = 0; w < kWays; ++w) {
                    const uint64_t wl = s0 + w * kWayWords;
                    mark_word(v.rs, wl + kKey0, v.gran_shift, last);
                    mark_word(v.rs, wl + kKey1, v.gran_shift, last);
                    if (w == target)
                        for (int q = 0; q < 4; ++q) mark_word(v.rs, wl + kVal + q, v.gran_shift, last);
                    mark_word(v.rs, wl + kLru, v.gran_shift, last);
                    mark_word(v.rs, wl + kFlags, v.gran_shift, last);
                }
                if (target < kWays) {
                    const uint64_t wl = s0 + target * kWayWords;
                    const uint32_t wmask = is_get ? (1u << kLru)
                                                  : (status == HETM_CACHE_UPDATED ? (0xfu << kVal) | (1u << kLru) : 0xffu);
                    uint64_t lw = ~0ull, lc = ~0ull;
#pragma unroll
                    for (int q = 0; q < kWayWords; ++q) {
                        if (!((wmask >> q) & 1u)) continue;
                        mark_word(v.ws, wl + q, v.gran_shift, lw);
                        mark_word(v.chunk, wl + q, v.chunk_shift, lc);
                    }
                    if (is_get) {
                        wlog_put(v, wbase, t, 0, (uint32_t)(wl + kLru));  // the LRU touch
                        wlog_put(v, wbase, t, 1, ~0u);
                    } else {
                        wlog_full = 1;  // up to 8 words: more than the log's 2 slots
                        wlog_put(v, wbase, t, 0, ~0u);
                        wlog_put(v, wbase, t, 1, ~0u);
                    }
                } else {
                    wlog_put(v, wbase, t, 0, ~0u);
                    wlog_put(v, wbase, t, 1, ~0u);
                }
                ++commits;
                break;
            }
            if (t != ~0ull) {  // aborted after taking a ticket: its log slots stay empty
                wlog_put(v, wbase, t, 0, ~0u);
                wlog_put(v, wbase, t, 1, ~0u);
            }
            ++aborts;
            if (block) {
                uint32_t ns = 32;
                for (int p = 0; p < 256 && ld_relaxed(lockp) == block; ++p) {
                    __nanosleep(ns);
                    ns = ns < 1024 ? 2 * ns : ns;
                }
            } else if (attempt >= 3) {  // hot set: jittered exponential backoff before re-reading it
                rng = rng * 6364136223846793005ull + 1442695040888963407ull;
                const uint32_t cap = 64u << (attempt < 8 ? attempt : 8);
                __nanosleep((uint32_t)(rng >> 40) % cap);
            }
            if (attempt >= max_attempts) {
                tickets[i] = ~0ull;
                ++livelocks;
                break;
            }
        }
    }
    if (__any_sync(0xffffffffu, wlog_full) && lane_id() == 0) ctr->wlog_overflow = 1;
    if (__any_sync(0xffffffffu, oob) && lane_id() == 0) atomicOr(&ctr->oob, 1u);
    commits = warp_sum(commits);
    aborts = warp_sum(aborts);
    livelocks = warp_sum(livelocks);
    if (lane_id() == 0) {
        if (commits) atomicAdd(&ctr->committed, commits);
        if (aborts) atomicAdd(&ctr->aborts, aborts);
        if (livelocks) atomicAdd(&ctr->livelocked, livelocks);
    }
}

cudaError_t launch_cache_batch(const ShardView& v, const CacheGeom& cg, const hetm_cache_tx* d_in, uint64_t n,
                               unsigned long long* d_tickets, hetm_cache_result* d_res, DevCounters* ctr,
                               uint32_t max_attempts, const LaunchGeom& g, cudaStream_t s) {
    if (n == 0) return cudaSuccess;
    uint64_t grid = (n + kCacheThreads - 1) / kCacheThreads;
    const uint64_t cap = (uint64_t)g.sm_count * 8;
    if (grid > cap) grid = cap;
    cache_batch_kernel<<<(unsigned)grid, kCacheThreads, 0, s>>>(v, cg, d_in, n, d_tickets, d_res, ctr, max_attempts);
    return cudaGetLastError();
}

}  // namespace hetm_b200
