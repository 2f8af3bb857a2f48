// tx_batch.cu — batch transaction kernels (guest-stm-batch).
//
// One launch executes a whole BatchSpec: thread i runs transaction i with
// priority i+1 (PR-STM priority rule, device_tm.cuh), retrying aborted
// attempts until commit or the livelock budget.  Commit
// fuses the RS/WS/ChunkMap instrumentation as fire-and-forget
// REDG.E.OR.64 and records the transaction's commit ticket.
#include <cstdlib>

#include "common.cuh"
#include "device_tm.cuh"
#include "kernels.h"
#include "phased_tx.cuh"

namespace hetm_b200 {

constexpr int kTxThreads = 256;

__device__ __forceinline__ void flush_batch_counters(unsigned long long commits, unsigned long long aborts,
                                                     unsigned long long livelocks, unsigned oob, DevCounters* ctr,
                                                     unsigned long long retried = 0) {
    retried = warp_sum(retried);
    if (lane_id() == 0 && retried) atomicAdd(&ctr->retried, retried);
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

// Bank transfer: read 4 accounts, acct0 -= amount, acct1 += amount.
// Warp-phased commit (phased_tx.cuh); each lane keeps its transaction across
// retries and moves to the next one (grid stride) once it commits.
//
// Contention management (zipf hot spots, BASELINE configs[2]).  The warp walks
// the commit phases in lock-step, so a lane must never wait in place for long:
//   * stopped by a FINAL holder: on the first attempts wait in place briefly
//     (the holder is mid-commit); later, SIT OUT — the lane polls that lock
//     word once per warp iteration and stays inactive until it changes, while
//     the other lanes keep committing;
//   * stopped by a version change (someone committed first), from the 4th
//     attempt: sit out a random 0..2^min(attempts-1, 6) iterations (up to 2^10
//     after 32 attempts), so the contenders of a hot word stop re-reading it in
//     lock-step (the ~N^2 wasted attempts of N contenders per hot word).
// Uniform access never gets here (0.4% aborts); zipf 0.8 over 2^27 accounts
// drops from 130 to 28 ms per 2^20-tx batch (profiles/r01_configs_probe.json).
template <int KO, int MINB = 4>
__global__ void __launch_bounds__(kTxThreads, MINB) bank_batch_kernel(ShardView v, const hetm_bank_tx* __restrict__ in,
                                                                   uint64_t n, unsigned long long* __restrict__ tickets,
                                                                   DevCounters* ctr, uint32_t max_attempts) {
    unsigned long long commits = 0, aborts = 0, livelocks = 0, retried = 0;
    unsigned oob = 0;
    uint64_t i, stride;
    tx_range(v, n, i, stride);
    uint32_t attempts = 0;
    bool loaded = false;
    uint64_t amount = 0;
    StaticTx<4, 2> tx;
    tx.block_lk = 0;
    uint32_t backoff = 0, block_polls = 0;
    unsigned long long rng = 0x9e3779b97f4a7c15ull * ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x + 1);
    unsigned long long clocks[6] = {0, 0, 0, 0, 0, 0};
    const unsigned long long wbase = ld_relaxed(&ctr->wlog_base);
    // the next record of this lane is fetched while the current one commits
    // (its DRAM round trip is off the per-transaction chain)
    uint64_t nx01 = 0, nx23 = 0, nxamt = 0;
    uint64_t nx_i = ~0ull;
    while (__any_sync(0xffffffffu, i < n)) {
        if (i < n && !loaded) {
            uint64_t w01, w23;
            if (nx_i == i) {
                w01 = nx01;
                w23 = nx23;
                amount = nxamt;
            } else {
                const uint64_t* rec = reinterpret_cast<const uint64_t*>(in + i);
                w01 = __ldg(rec);
                w23 = __ldg(rec + 1);
                amount = __ldg(rec + 2);
            }
            if (i + stride < n) {
                const uint64_t* nrec = reinterpret_cast<const uint64_t*>(in + i + stride);
                nx01 = __ldg(nrec);
                nx23 = __ldg(nrec + 1);
                nxamt = __ldg(nrec + 2);
                nx_i = i + stride;
            }
            const uint64_t l0 = (w01 & 0xffffffffu) - v.base, l1 = (w01 >> 32) - v.base;
            const uint64_t l2 = (w23 & 0xffffffffu) - v.base, l3 = (w23 >> 32) - v.base;
            if (l0 >= v.size_words || l1 >= v.size_words || l2 >= v.size_words || l3 >= v.size_words) {
                tickets[i] = ~0ull;  // outside this shard: rejected, reported as OutOfBounds
                oob = 1;
                i += stride;
            } else {
                tx.loc[0] = (uint32_t)l0;
                tx.loc[1] = (uint32_t)l1;
                tx.loc[2] = (uint32_t)l2;
                tx.loc[3] = (uint32_t)l3;
                tx.first = first_occurrences(tx.loc);
                if constexpr ((KO & KO_STRIPES) != 0) {
#pragma unroll
                    for (int k = 0; k < 4; ++k) tx.sidx[k] = stripe_of(tx.loc[k], v.stripe_shift);
                    tx.sfirst = first_occurrences(tx.sidx);
                }
                loaded = true;
            }
        }
        // A lane whose last attempt was stopped by a FINAL holder sits out (one
        // poll of that word per warp iteration) until the holder releases it,
        // so the other lanes of the warp keep committing meanwhile.
        bool blocked = false;
        if (i < n && loaded && tx.block_lk) {
            blocked = lock_value<KO>(v, tx.block_loc) == tx.block_lk;
            // bounded: the same lock word can come back (a holder that aborted and
            // re-locked with the same priority and version), so after 256 polls the
            // lane simply tries again
            if (blocked && ++block_polls > 256) blocked = false;
            if (!blocked) {
                tx.block_lk = 0;
                block_polls = 0;
            }
        }
        if (i < n && loaded && backoff) {  // randomized sit-out after repeated version-change aborts
            --backoff;
            blocked = true;
        }
        if (__all_sync(0xffffffffu, blocked || !(i < n && loaded))) __nanosleep(256);  // whole warp waits
        const bool active = i < n && loaded && !blocked;
        unsigned long long t = ~0ull;
        const auto transfer = [&](StaticTx<4, 2>& x) {
            x.wval[0] = x.val[0] - amount;
            x.wval[1] = x.val[1] + amount;
        };
        bool committed;
        if constexpr ((KO & KO_STRIPES) != 0)
            committed = striped_attempt<4, 2, KO>(tx, active, (uint32_t)(i + 1), v, &ctr->ticket, t, transfer);
        else
            committed = phased_attempt<4, 2, KO>(tx, active, (uint32_t)(i + 1), v, &ctr->ticket, t, transfer, clocks);
        if (committed) {
            tickets[i] = t;
            if constexpr ((KO & KO_TRACE) != 0) {  // reads acct0..3 in order, then writes acct0, acct1
                unsigned long long* r = v.trace + i * kTraceWords;
                r[0] = t;
                r[1] = tx.val[0];
                r[2] = tx.val[1];
                r[3] = tx.rv[0];
                r[4] = tx.rv[1];
                r[5] = tx.val[0];
                r[6] = tx.val[1];
                r[7] = tx.wval[0];
                r[8] = tx.wval[1];
            }
            wlog_put(v, wbase, t, 0, tx.loc[0]);
            wlog_put(v, wbase, t, 1, tx.loc[1]);
            ++commits;
            retried += attempts >= 2;
        } else if (active) {
            if (t != ~0ull) {  // aborted after taking a ticket: its log slots stay empty
                wlog_put(v, wbase, t, 0, ~0u);
                wlog_put(v, wbase, t, 1, ~0u);
            }
            ++aborts;
            // mild contention: the holder is mid-commit, wait in place briefly (cell
            // locks; a stripe is mostly held by a transaction on ANOTHER word of
            // it, so the lane sits out at once)
            if ((KO & KO_STRIPES) == 0 && tx.block_lk && attempts < 4) {
                uint32_t ns = 32;
                for (int p = 0; p < 16 && lock_value<KO>(v, tx.block_loc) == tx.block_lk; ++p) {
                    __nanosleep(ns);
                    ns = ns < 512 ? 2 * ns : ns;
                }
                tx.block_lk = 0;
            }
            if (!tx.block_lk && attempts >= 4) {  // hot word: spread the retries over 2^min(attempts-1, 6 / 10 from 32) iterations
                rng = rng * 6364136223846793005ull + 1442695040888963407ull;
                backoff = (uint32_t)(rng >> 40) & ((1u << (attempts < 7 ? attempts - 1 : (attempts < 32 ? 6 : 10))) - 1u);
            }
            if (++attempts < max_attempts) continue;
            tickets[i] = ~0ull;
            ++livelocks;
        } else {
            continue;
        }
        i += stride;
        loaded = false;
        attempts = 0;
        tx.block_lk = 0;
        backoff = 0;
    }
    if constexpr ((KO & KO_COUNT_TICKETS) != 0) {
        const unsigned long long x = warp_sum(clocks[0]);
        if (lane_id() == 0) atomicAdd(&ctr->pad[4], x);
    }
    if constexpr ((KO & KO_PHASE_CLOCKS) != 0) {
#pragma unroll
        for (int p = 0; p < 6; ++p) {
            const unsigned long long x = warp_sum(clocks[p]);
            if (lane_id() == 0) atomicAdd(&ctr->pad[p], x);
        }
    }
    flush_batch_counters(commits, aborts, livelocks, oob, ctr, retried);
}

// Generic <=4 reads / <=2 read-modify-writes (hetm_rw_tx) through the
// TM_read / TM_write / TM_commit interface of device_tm.cuh.
__global__ void __launch_bounds__(kTxThreads) rw_batch_kernel(ShardView v, const hetm_rw_tx* __restrict__ in, uint64_t n,
                                                              unsigned long long* __restrict__ tickets,
                                                              DevCounters* ctr, uint32_t max_attempts) {
    unsigned long long commits = 0, aborts = 0, livelocks = 0;
    unsigned oob = 0;
    const unsigned long long wbase = ld_relaxed(&ctr->wlog_base);
    uint64_t i0, stride;
    tx_range(v, n, i0, stride);
    for (uint64_t i = i0; i < n; i += stride) {
        const hetm_rw_tx r = in[i];
        const uint32_t nr = r.nr < 4 ? r.nr : 4, nw = r.nw < 2 ? r.nw : 2;
        bool in_shard = true;
        for (uint32_t j = 0; j < nr; ++j) in_shard &= (r.r_addr[j] - v.base) < v.size_words;
        for (uint32_t j = 0; j < nw; ++j) in_shard &= (r.w_addr[j] - v.base) < v.size_words;
        if (!in_shard) {
            tickets[i] = ~0ull;
            oob = 1;
            continue;
        }
        DeviceTx<6, 2> tx;
        uint32_t attempt = 0;
        for (;;) {
            ++attempt;
            tx.begin((uint32_t)(i + 1));
            bool ok = true;
            uint64_t sum = 0;
            uint64_t rx[4] = {0, 0, 0, 0}, cx[2] = {0, 0}, wx[2] = {0, 0};  // trace: values in program order
            for (uint32_t j = 0; j < nr && ok; ++j) {
                uint64_t x;
                ok = tm_read(tx, v, r.r_addr[j] - v.base, x);
                rx[j] = x;
                sum += x;
            }
            for (uint32_t j = 0; j < nw && ok; ++j) {
                uint64_t cur;
                const uint64_t loc = r.w_addr[j] - v.base;
                ok = tm_read(tx, v, loc, cur) && tm_write(tx, v, loc, cur + r.add[j] + sum);
                cx[j] = cur;
                wx[j] = cur + r.add[j] + sum;
            }
            unsigned long long t = ~0ull;
            if (ok && tm_commit(tx, v, &ctr->ticket, t)) {
                tickets[i] = t;
                if (v.trace) {
                    unsigned long long* tr = v.trace + i * kTraceWords;
                    tr[0] = t;
                    for (int j = 0; j < 4; ++j) tr[1 + j] = rx[j];
                    for (int j = 0; j < 2; ++j) {
                        tr[5 + j] = cx[j];
                        tr[7 + j] = wx[j];
                    }
                }
                tm_mark_bitmaps(tx, v);
                wlog_put(v, wbase, t, 0, tx.nw > 0 ? (uint32_t)tx.w_local[0] : ~0u);
                wlog_put(v, wbase, t, 1, tx.nw > 1 ? (uint32_t)tx.w_local[1] : ~0u);
                ++commits;
                break;
            }
            if (t != ~0ull) {  // aborted after taking a ticket: its log slots stay empty
                wlog_put(v, wbase, t, 0, ~0u);
                wlog_put(v, wbase, t, 1, ~0u);
            }
            ++aborts;
            if (attempt >= 4) __nanosleep(attempt < 64 ? 32u * attempt : 2048u);
            if (attempt >= max_attempts) {
                tickets[i] = ~0ull;
                ++livelocks;
                break;
            }
        }
    }
    flush_batch_counters(commits, aborts, livelocks, oob, ctr);
}

static unsigned grid_for(uint64_t n, int threads, int blocks_per_sm, int sms) {
    uint64_t want = (n + threads - 1) / threads;
    uint64_t cap = (uint64_t)blocks_per_sm * (uint64_t)sms;
    if (want > cap) want = cap;
    return (unsigned)(want ? want : 1);
}

cudaError_t launch_bank_batch(const ShardView& v, const hetm_bank_tx* d_in, uint64_t n, unsigned long long* d_tickets,
                              DevCounters* ctr, uint32_t max_attempts, const LaunchGeom& g, cudaStream_t s) {
    if (n == 0) return cudaSuccess;
#ifdef HETM_EXPERIMENTS
    static const int ko = [] {  // phase knockouts (make EXPERIMENTS=1): profiling only, some incorrect
        const char* e = std::getenv("HETM_KNOCKOUT");
        return e ? std::atoi(e) : 0;
    }();
#endif
    static const int bps = [] {  // occupancy experiments only
        const char* e = std::getenv("HETM_TX_BLOCKS_PER_SM");
        return e ? std::atoi(e) : 0;
    }();
    const unsigned grid = grid_for(n, kTxThreads, bps > 0 ? bps : g.max_blocks_tx, g.sm_count);
#define HETM_KO_CASE(K) \
    case K: bank_batch_kernel<K><<<grid, kTxThreads, 0, s>>>(v, d_in, n, d_tickets, ctr, max_attempts); break;
    if (v.trace) {  // checker traces: the KO_TRACE instantiation (the product one is untouched)
        if (v.stripes)
            bank_batch_kernel<KO_TRACE | KO_STRIPES, 2><<<grid, kTxThreads, 0, s>>>(v, d_in, n, d_tickets, ctr, max_attempts);
        else
            bank_batch_kernel<KO_TRACE><<<grid, kTxThreads, 0, s>>>(v, d_in, n, d_tickets, ctr, max_attempts);
        return cudaGetLastError();
    }
    static const int spin = [] {  // tuning experiments: HETM_STRIPE_SPIN=1 waits for P0 holders
        const char* e = std::getenv("HETM_STRIPE_SPIN");
        return e ? std::atoi(e) : 0;
    }();
#ifdef HETM_EXPERIMENTS
    static const int sko = [] {  // stripe-kernel phase knockouts (make EXPERIMENTS=1): profiling only, incorrect
        const char* e = std::getenv("HETM_STRIPE_KO");
        return e ? std::atoi(e) : 0;
    }();
    if (v.stripes && sko) {
        constexpr int S = KO_STRIPES;
        switch (sko) {
            case KO_BITMAPS: bank_batch_kernel<S | KO_BITMAPS, 2><<<grid, kTxThreads, 0, s>>>(v, d_in, n, d_tickets, ctr, max_attempts); break;
            case KO_NO_TICKET: bank_batch_kernel<S | KO_NO_TICKET, 2><<<grid, kTxThreads, 0, s>>>(v, d_in, n, d_tickets, ctr, max_attempts); break;
            case KO_SKIP_VALIDATE: bank_batch_kernel<S | KO_SKIP_VALIDATE, 2><<<grid, kTxThreads, 0, s>>>(v, d_in, n, d_tickets, ctr, max_attempts); break;
            case KO_NO_FENCE: bank_batch_kernel<S | KO_NO_FENCE, 2><<<grid, kTxThreads, 0, s>>>(v, d_in, n, d_tickets, ctr, max_attempts); break;
            default: bank_batch_kernel<S | KO_BITMAPS | KO_NO_TICKET | KO_SKIP_VALIDATE | KO_NO_FENCE, 2><<<grid, kTxThreads, 0, s>>>(v, d_in, n, d_tickets, ctr, max_attempts);
        }
        return cudaGetLastError();
    }
#endif
    static const int two_pl = [] {  // tuning experiments: HETM_STRIPE_2PL=1 locks the read-only stripes too
        const char* e = std::getenv("HETM_STRIPE_2PL");
        return e ? std::atoi(e) : 0;
    }();
    if (v.stripes && two_pl) {
        bank_batch_kernel<KO_STRIPES | KO_STRIPE_2PL, 2><<<grid, kTxThreads, 0, s>>>(v, d_in, n, d_tickets, ctr,
                                                                                    max_attempts);
        return cudaGetLastError();
    }
    if (v.stripes) {  // product: lock words in the L2-resident stripe table
        if (spin)
            bank_batch_kernel<KO_STRIPES | KO_STRIPE_SPIN, 2><<<grid, kTxThreads, 0, s>>>(v, d_in, n, d_tickets, ctr,
                                                                                         max_attempts);
        else
            bank_batch_kernel<KO_STRIPES, 2><<<grid, kTxThreads, 0, s>>>(v, d_in, n, d_tickets, ctr, max_attempts);
        return cudaGetLastError();
    }
#ifdef HETM_EXPERIMENTS
    switch (ko) {
        HETM_KO_CASE(4) HETM_KO_CASE(8) HETM_KO_CASE(16) HETM_KO_CASE(64) HETM_KO_CASE(128) HETM_KO_CASE(256) HETM_KO_CASE(512) HETM_KO_CASE(1024) HETM_KO_CASE(1536)
        default: bank_batch_kernel<0><<<grid, kTxThreads, 0, s>>>(v, d_in, n, d_tickets, ctr, max_attempts);
    }
#else
    bank_batch_kernel<0><<<grid, kTxThreads, 0, s>>>(v, d_in, n, d_tickets, ctr, max_attempts);
#endif
#undef HETM_KO_CASE
    return cudaGetLastError();
}

cudaError_t launch_rw_batch(const ShardView& v, const hetm_rw_tx* d_in, uint64_t n, unsigned long long* d_tickets,
                            DevCounters* ctr, uint32_t max_attempts, const LaunchGeom& g, cudaStream_t s) {
    if (n == 0) return cudaSuccess;
    rw_batch_kernel<<<grid_for(n, kTxThreads, g.max_blocks_tx, g.sm_count), kTxThreads, 0, s>>>(v, d_in, n, d_tickets,
                                                                                                ctr, max_attempts);
    return cudaGetLastError();
}

int query_tx_occupancy(int* bank_blocks) {
    int b = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, bank_batch_kernel<0>, kTxThreads, 0) != cudaSuccess)
        return -1;
    *bank_blocks = b;
    return 0;
}

}  // namespace hetm_b200
