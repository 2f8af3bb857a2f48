// bank_sched.cu — the SCAN schedule of the bank batch: a skew-proof,
// abort-free execution of a whole batch in input order (ticket = first + i).
//
// A bank transaction's writes are read-modify-writes with known deltas
// (acct0 -= amount, acct1 += amount; acct2/acct3 only read), so the serial
// execution of the batch in input order is a per-account sum of deltas:
//   1. per transaction (coalesced): one 32-bit key per written account with
//      the payload (2 i + k) << 1 | writer and the access's delta (the tx's
//      net effect on the account: last write wins when acct0 == acct1, whose
//      second slot is then dropped), and the RS bits of the read-only
//      accounts (probe-gated, per-CTA filter); the ticket and write-set log
//      slots are written here too;
//   2. radix sort of the 2n (account, payload) pairs on the account bits
//      only (sort.cu, hand-written: 3 passes of <= 10-bit digits) — the sort
//      is stable, so each account's accesses stay in input order;
//   3. one pass over the sorted accesses (sched_commit_red_kernel): per warp
//      run a segmented shuffle sum of the deltas, added to the cell with one
//      RED.ADD (commutative: a hot account spread over many runs needs no
//      order); at each account's segment end the version of its last writer
//      (lk_commit of its ticket) is stored; RS / WS / ChunkMap bits are set
//      warp-aggregated (the stream is sorted).
// A traced batch keys all four accesses ((4 i + k) << 1 | writer), runs an
// inclusive scan-by-account of {delta, last writer} (sort.cu), records every access's
// pre-value (sched_trace_kernel) and commits from the scan (sched_commit_kernel).
// Cost is independent of skew (no locks, no retries): at zipf 0.99 the
// optimistic PR-STM kernel serializes ~10^5 commits on the hottest account.
// The result is exactly the deterministic single-worker mode.
#include "common.cuh"
#include "device_tm.cuh"
#include "kernels.h"

#include <algorithm>
#include <cstring>
#include <vector>

namespace hetm_b200 {

namespace {

constexpr unsigned kSchedThreads = 256;
constexpr unsigned long long kNone = ~0ull;
constexpr uint32_t kNoLoc = 0xffffffffu;  // sort sentinel: accesses of rejected transactions
constexpr unsigned kSeenLog = 11, kSeenSlots = 1u << kSeenLog;  // keys kernel: per-CTA RS filter (16 KiB)
constexpr int kCommitU = 4;                                      // commit kernel: 32-access runs per warp sweep
constexpr int kKeysU = 2;                                        // keys kernel: transactions per thread per sweep

struct DeltaW {  // scan value: summed delta, last writing transaction (input index) or kNone
    unsigned long long d, w;
};
// Sort payload: access index a = S i + k (input order) << 1 | writer, where
// writer marks the transaction's first slot naming an account it writes and S
// is the slots keyed per transaction (2: the written accounts; 4: all, traced).
__device__ __forceinline__ uint32_t acc_of(uint32_t p) { return p >> 1; }
template <int S>
__device__ __forceinline__ uint64_t tx_of(uint32_t p) { return p >> (S == 4 ? 3 : 2); }

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

// Per transaction (coalesced): the S sort keys + payloads, the per-access
// deltas (the tx's net effect on an account — the last write wins, acct1
// after acct0 — on the first slot naming it), its ticket and write-set log
// slots, and (S = 2) the RS bits of its read-only accounts; a rejected
// (out-of-shard) transaction gets sentinel keys, no ticket, no bits and empty
// log slots.
template <int S>
__global__ void sched_keys_kernel(ShardView v, const hetm_bank_tx* __restrict__ in, uint64_t n,
                                  uint32_t* __restrict__ locs, uint32_t* __restrict__ pay,
                                  unsigned long long* __restrict__ delta, unsigned long long* __restrict__ tickets,
                                  const unsigned long long* first, DevCounters* ctr) {
    // RS bits this CTA already set (hashed by bit, the full bit index stored:
    // a hit is exact): hot read-only accounts of a skewed batch then cost one
    // atomic per CTA instead of a queue of them on cleared bitmaps.
    __shared__ unsigned long long seen[kSeenSlots];
    if (S == 2) {
        for (unsigned q = threadIdx.x; q < kSeenSlots; q += blockDim.x) seen[q] = ~0ull;
        __syncthreads();
    }
    const unsigned long long t0 = *first, wbase = ld_relaxed(&ctr->wlog_base);
    unsigned oob = 0;
    unsigned long long commits = 0;
    // kKeysU transactions per thread per sweep, their records loaded up front
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t i0 = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i0 < n; i0 += stride * kKeysU) {
        uint64_t aa[kKeysU][4], am[kKeysU];
#pragma unroll
        for (int u = 0; u < kKeysU; ++u)
            if (i0 + u * stride < n) load_accts(in, i0 + u * stride, v.base, aa[u], am[u]);
#pragma unroll
        for (int u = 0; u < kKeysU; ++u) {
            const uint64_t i = i0 + u * stride;
            if (i >= n) break;
            const uint64_t(&a)[4] = aa[u];
            const uint64_t amount = am[u];
            const bool ok = a[0] < v.size_words && a[1] < v.size_words && a[2] < v.size_words && a[3] < v.size_words;
            if (S == 2 && ok) {  // RS of the read-only accounts (the sorted written ones: commit kernel)
#pragma unroll
                for (int k = 2; k < 4; ++k) {
                    const uint64_t b = a[k] >> v.gran_shift;
                    unsigned long long* slot = &seen[(b * 0x9e3779b97f4a7c15ull) >> (64 - kSeenLog)];
                    if (a[k] != a[0] && a[k] != a[1] && atomicAdd(slot, 0ull) != b) {  // one 64-bit word: exact
                        if (!test_bit(v.rs, b)) set_bit(v.rs, b);
                        atomicExch(slot, b);
                    }
                }
            }
            const unsigned long long t = t0 + i;
            oob |= !ok;
            commits += ok;
            tickets[i] = ok ? t : kNone;
            wlog_put(v, wbase, t, 0, ok ? (uint32_t)a[0] : ~0u);
            wlog_put(v, wbase, t, 1, ok ? (uint32_t)a[1] : ~0u);
#pragma unroll
            for (int k = 0; k < S; ++k) {
                bool first_slot = true;
#pragma unroll
                for (int q = 0; q < k; ++q) first_slot &= a[q] != a[k];
                const unsigned long long d = !first_slot ? 0ull : a[k] == a[1] ? amount : a[k] == a[0] ? 0ull - amount : 0ull;
                const bool writer = first_slot && (a[k] == a[0] || a[k] == a[1]);
                // S = 2: slot 1 of a transfer onto its own account is dropped, so every
                // live sorted access is a writer (the reduction commit relies on it)
                locs[S * i + k] = ok && (S == 4 || first_slot) ? (uint32_t)a[k] : kNoLoc;
                pay[S * i + k] = (uint32_t)(S * i + k) << 1 | (uint32_t)writer;
                delta[S * i + k] = d;
            }
        }
    }
    if (__any_sync(0xffffffffu, oob) && lane_id() == 0) atomicOr(&ctr->oob, 1u);
    const unsigned long long c = warp_sum(commits);
    if (lane_id() == 0 && c) atomicAdd(&ctr->committed, c);
}

// First ticket of the batch (ticket = first + input index).
__global__ void sched_ticket_kernel(DevCounters* ctr, uint64_t n, unsigned long long* first) {
    *first = atomicAdd(&ctr->ticket, (unsigned long long)n);
}

// Read-only pass (traced batches): the value every access reads = the account's
// batch-start value + the deltas of the earlier transactions.
__global__ void sched_trace_kernel(ShardView v, const hetm_bank_tx* __restrict__ in, uint64_t n4,
                                   const uint32_t* __restrict__ locs, const uint32_t* __restrict__ pay,
                                   const unsigned long long* __restrict__ delta, const DeltaW* __restrict__ incl,
                                   const unsigned long long* first) {
    const unsigned long long t0 = *first;
    for (uint64_t j = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; j < n4; j += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t loc = locs[j];
        if (loc == kNoLoc) continue;
        const uint64_t i = tx_of<4>(pay[j]);
        const int k = (int)(acc_of(pay[j]) & 3);
        // pre-value: exclusive of this transaction's own delta, which sits on its
        // first slot naming the account (this entry or an earlier one of tx i)
        uint64_t jj = j;
        while (jj > 0 && locs[jj - 1] == loc && tx_of<4>(pay[jj - 1]) == i) --jj;
        const unsigned long long pre = v.cells[loc].value + incl[jj].d - delta[acc_of(pay[jj])];
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

// Per sorted access: RS at each account's first access, the final value and
// version + WS / ChunkMap at its last one if the account was written.  A warp
// walks 32 consecutive sorted accesses, so its bitmap bits arrive in word
// order: each run of lanes on one bitmap word issues a single probe-gated
// atomic (the first batch of a round, on cleared bitmaps, otherwise queues
// thousands of atomics on the words of hot accounts).
template <int S>
__global__ void sched_commit_kernel(ShardView v, uint64_t n4, const uint32_t* __restrict__ locs,
                                    const DeltaW* __restrict__ incl, const unsigned long long* first) {
    // A warp takes kCommitU consecutive 32-access runs per sweep and issues each
    // stage's loads for all of them before using any (memory-level parallelism:
    // the stages are dependent — account, then scan value, then cell).
    constexpr int U = kCommitU;
    const unsigned long long t0 = *first;
    const unsigned lane = lane_id();
    const uint64_t sweep = (uint64_t)gridDim.x * blockDim.x * U;
    for (uint64_t base = ((uint64_t)blockIdx.x * blockDim.x + (threadIdx.x & ~31u)) * U; base < n4; base += sweep) {
        uint32_t loc[U];
        bool seg_first[U], seg_last[U], wrote[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const uint64_t j = base + (uint64_t)u * 32 + lane;
            loc[u] = j < n4 ? locs[j] : kNoLoc;
            const uint32_t prev = j > 0 && j - 1 < n4 ? locs[j - 1] : kNoLoc;
            const uint32_t next = j + 1 < n4 ? locs[j + 1] : kNoLoc;
            seg_first[u] = loc[u] != kNoLoc && (j == 0 || prev != loc[u]);
            seg_last[u] = loc[u] != kNoLoc && next != loc[u];
        }
        DeltaW x[U];
#pragma unroll
        for (int u = 0; u < U; ++u) x[u] = seg_last[u] ? incl[base + (uint64_t)u * 32 + lane] : DeltaW{0, kNone};
        uint64_t val[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            wrote[u] = x[u].w != kNone;
            val[u] = wrote[u] ? v.cells[loc[u]].value : 0;
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            if (wrote[u]) st_pair(&v.cells[loc[u]], val[u] + x[u].d, lk_commit(t0 + x[u].w));
            warp_set_bits_sorted(v.rs, (uint64_t)loc[u] >> v.gran_shift, seg_first[u]);  // every access reads
            warp_set_bits_sorted(v.ws, (uint64_t)loc[u] >> v.gran_shift, wrote[u]);
            warp_set_bits_sorted(v.chunk, (uint64_t)loc[u] >> v.chunk_shift, wrote[u]);
        }
    }
}

// The untraced commit (S = 2, every live access a writer): no scan.  A
// warp takes 32 consecutive sorted accesses (kCommitU runs per sweep); a
// segmented prefix sum over the run's lanes (runs of one account are
// contiguous: the stream is sorted) leaves each run's delta total on its last
// lane, which adds it to the cell's value with one fire-and-forget RED.ADD —
// addition commutes, so an account split over several runs (a hot account of
// a skewed batch) needs no ordering between them — and, if the run ends the
// account's segment, stores the version of the last writer (the stable sort
// keeps input order, so that is the segment's last access).  No load of the
// cell: the serial input-order result is value + sum of deltas.
__global__ void sched_commit_red_kernel(ShardView v, uint64_t n2, const uint32_t* __restrict__ locs,
                                        const uint32_t* __restrict__ pay, const unsigned long long* __restrict__ delta,
                                        const unsigned long long* first) {
    constexpr int U = kCommitU;
    const unsigned long long t0 = *first;
    const unsigned lane = lane_id();
    const uint64_t sweep = (uint64_t)gridDim.x * blockDim.x * U;
    for (uint64_t base = ((uint64_t)blockIdx.x * blockDim.x + (threadIdx.x & ~31u)) * U; base < n2; base += sweep) {
        uint32_t loc[U], p[U];
        bool seg_first[U], seg_last[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const uint64_t j = base + (uint64_t)u * 32 + lane;
            loc[u] = j < n2 ? locs[j] : kNoLoc;
            p[u] = j < n2 ? pay[j] : 0u;
            const uint32_t prev = j > 0 && j - 1 < n2 ? locs[j - 1] : kNoLoc;
            const uint32_t next = j + 1 < n2 ? locs[j + 1] : kNoLoc;
            seg_first[u] = loc[u] != kNoLoc && (j == 0 || prev != loc[u]);
            seg_last[u] = loc[u] != kNoLoc && next != loc[u];
        }
        unsigned long long d[U];
#pragma unroll
        for (int u = 0; u < U; ++u) d[u] = loc[u] != kNoLoc ? delta[acc_of(p[u])] : 0ull;
#pragma unroll
        for (int u = 0; u < U; ++u) {
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {  // segmented inclusive prefix sum within the run
                const uint32_t lo = __shfl_up_sync(0xffffffffu, loc[u], o);
                const unsigned long long dd = __shfl_up_sync(0xffffffffu, d[u], o);
                if (lane >= (unsigned)o && lo == loc[u]) d[u] += dd;
            }
            const uint32_t nxt = __shfl_down_sync(0xffffffffu, loc[u], 1);
            const bool run_last = loc[u] != kNoLoc && (lane == 31 || nxt != loc[u]);
            if (run_last) {
                Cell* c = &v.cells[loc[u]];
                if (d[u]) atomicAdd(reinterpret_cast<unsigned long long*>(&c->value), d[u]);  // RED.E.ADD.64
                if (seg_last[u]) st_relaxed(&c->meta, lk_commit(t0 + tx_of<2>(p[u])));
            }
            warp_set_bits_sorted(v.rs, (uint64_t)loc[u] >> v.gran_shift, seg_first[u]);  // every access reads
            warp_set_bits_sorted(v.ws, (uint64_t)loc[u] >> v.gran_shift, seg_last[u]);
            warp_set_bits_sorted(v.chunk, (uint64_t)loc[u] >> v.chunk_shift, seg_last[u]);
        }
    }
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
    const int end_bit = (int)std::min<uint32_t>(32, bits_for(size_words) + 1);  // + the sentinel
    auto al = [](size_t x) { return (x + 255) & ~size_t(255); };
    // [locs in/out | payload in/out | delta | scan | first ticket | sort / scan temp]
    return 4 * al(n4 * 4) + al(n4 * 8) + al(n4 * sizeof(DeltaW)) + 256 +
           al(std::max(radix_sort_temp_bytes(n4, end_bit), seg_scan_temp_bytes(n4)));
}

cudaError_t launch_bank_sched(const ShardView& v, const hetm_bank_tx* d_in, uint64_t n, unsigned long long* d_tickets,
                              DevCounters* ctr, void* temp, size_t temp_bytes, const LaunchGeom& g, cudaStream_t s,
                              SchedGraph* graph) {
    if (n == 0) return cudaSuccess;
    if (cudaError_t e = radix_sort_init(); e != cudaSuccess) return e;  // before any capture
    if (graph && !v.trace) {
        // Replay the captured sequence: ~12 dependent launches (3 sort passes of
        // 3 kernels each) cost more host time than GPU time when issued
        // one by one.  Only the keys kernel's inputs / tickets change per batch.
        const bool same = graph->exec && graph->n == n && graph->temp == temp && graph->wlog == v.wlog &&
                          graph->wlog_slots == v.wlog_slots && graph->cells == v.cells && graph->ctr == ctr;
        if (!same) {
            if (graph->exec) cudaGraphExecDestroy(graph->exec);
            if (graph->graph) cudaGraphDestroy(graph->graph);
            graph->exec = nullptr;
            graph->graph = nullptr;
            if (!graph->cap) {
                cudaError_t e = cudaStreamCreateWithFlags(&graph->cap, cudaStreamNonBlocking);
                if (e != cudaSuccess) return e;
            }
            cudaError_t e = cudaStreamBeginCapture(graph->cap, cudaStreamCaptureModeThreadLocal);
            if (e != cudaSuccess) return e;
            e = launch_bank_sched(v, d_in, n, d_tickets, ctr, temp, temp_bytes, g, graph->cap, nullptr);
            cudaGraph_t gr = nullptr;
            const cudaError_t e2 = cudaStreamEndCapture(graph->cap, &gr);
            if (e != cudaSuccess || e2 != cudaSuccess) {
                if (gr) cudaGraphDestroy(gr);
                return e != cudaSuccess ? e : e2;
            }
            size_t nn = 0;
            cudaGraphGetNodes(gr, nullptr, &nn);
            std::vector<cudaGraphNode_t> nodes(nn);
            cudaGraphGetNodes(gr, nodes.data(), &nn);
            graph->keys_node = nullptr;
            for (auto nd : nodes) {
                cudaGraphNodeType t;
                cudaKernelNodeParams kp{};
                if (cudaGraphNodeGetType(nd, &t) == cudaSuccess && t == cudaGraphNodeTypeKernel &&
                    cudaGraphKernelNodeGetParams(nd, &kp) == cudaSuccess &&
                    kp.func == reinterpret_cast<void*>(sched_keys_kernel<2>)) {
                    graph->keys_node = nd;
                    auto& a = graph->keys_args;
                    void* dst[9] = {&a.v, &a.in, &a.n, &a.locs, &a.pay, &a.delta, &a.tickets, &a.first, &a.ctr};
                    const size_t sz[9] = {sizeof a.v, 8, 8, 8, 8, 8, 8, 8, 8};
                    for (int q = 0; q < 9; ++q) {
                        std::memcpy(dst[q], kp.kernelParams[q], sz[q]);
                        graph->keys_ptrs[q] = dst[q];
                    }
                    graph->keys_params = kp;
                    graph->keys_params.kernelParams = graph->keys_ptrs;
                    graph->keys_params.extra = nullptr;
                }
            }
            e = graph->keys_node ? cudaGraphInstantiate(&graph->exec, gr, 0) : cudaErrorUnknown;
            if (e != cudaSuccess) {
                cudaGraphDestroy(gr);
                graph->exec = nullptr;
                return e;
            }
            graph->graph = gr;
            graph->n = n;
            graph->temp = temp;
            graph->wlog = v.wlog;
            graph->wlog_slots = v.wlog_slots;
            graph->cells = v.cells;
            graph->ctr = ctr;
        }
        // sched_keys_kernel(v, in, n, locs, pay, delta, tickets, first, ctr): patch in + tickets
        if (graph->keys_args.in != d_in || graph->keys_args.tickets != d_tickets) {
            graph->keys_args.in = d_in;
            graph->keys_args.tickets = d_tickets;
            cudaError_t e = cudaGraphExecKernelNodeSetParams(graph->exec, graph->keys_node, &graph->keys_params);
            if (e != cudaSuccess) return e;
        }
        return cudaGraphLaunch(graph->exec, s);
    }
    // keyed slots: the two written accounts, or all four accesses for a trace
    const int S = v.trace ? 4 : 2;
    if ((uint64_t)S * n * 2 > (1ull << 32)) return cudaErrorInvalidValue;  // (S*i + k) << 1 payloads fit 32 bits
    const uint64_t n4 = (uint64_t)S * n;
    const int end_bit = (int)std::min<uint32_t>(32, bits_for(v.size_words) + 1);
    auto al = [](size_t x) { return (x + 255) & ~size_t(255); };
    char* p = static_cast<char*>(temp);
    uint32_t* locs = reinterpret_cast<uint32_t*>(p);
    uint32_t* locs_s = reinterpret_cast<uint32_t*>(p + al(n4 * 4));
    uint32_t* pay = reinterpret_cast<uint32_t*>(p + 2 * al(n4 * 4));
    uint32_t* pay_s = reinterpret_cast<uint32_t*>(p + 3 * al(n4 * 4));
    auto* delta = reinterpret_cast<unsigned long long*>(p + 4 * al(n4 * 4));
    auto* incl = reinterpret_cast<DeltaW*>(p + 4 * al(n4 * 4) + al(n4 * 8));
    const size_t off = 4 * al(n4 * 4) + al(n4 * 8) + al(n4 * sizeof(DeltaW));
    auto* first = reinterpret_cast<unsigned long long*>(p + off);
    void* sort_tmp = p + off + 256;
    const size_t sort_bytes = temp_bytes - (off + 256);
    const unsigned grid_tx = grid_for(n, kSchedThreads, 8, g.sm_count);
    const unsigned grid_acc = grid_for(n4, kSchedThreads, 8, g.sm_count);
    sched_ticket_kernel<<<1, 1, 0, s>>>(ctr, n, first);
    if (S == 4) sched_keys_kernel<4><<<grid_tx, kSchedThreads, 0, s>>>(v, d_in, n, locs, pay, delta, d_tickets, first, ctr);
    else sched_keys_kernel<2><<<grid_tx, kSchedThreads, 0, s>>>(v, d_in, n, locs, pay, delta, d_tickets, first, ctr);
    cudaError_t e = radix_sort_pairs(locs, locs_s, pay, pay_s, n4, end_bit, sort_tmp, sort_bytes, g, s);
    if (e != cudaSuccess) return e;
    if (S == 4) {
        e = seg_scan_delta_writer(locs_s, pay_s, delta, n4, reinterpret_cast<unsigned long long*>(incl), sort_tmp,
                                  sort_bytes, s);
        if (e != cudaSuccess) return e;
        sched_trace_kernel<<<grid_acc, kSchedThreads, 0, s>>>(v, d_in, n4, locs_s, pay_s, delta, incl, first);
        sched_commit_kernel<4><<<grid_acc, kSchedThreads, 0, s>>>(v, n4, locs_s, incl, first);
    } else {
        sched_commit_red_kernel<<<grid_acc, kSchedThreads, 0, s>>>(v, n4, locs_s, pay_s, delta, first);
    }
    return cudaGetLastError();
}

}  // namespace hetm_b200
