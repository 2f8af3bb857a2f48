// gen.cpp — seeded host-side input generators (bank batches, host write logs).
//
// Deterministic generator per det_rng.hpp:8-42 (splitmix64 state walk, Lemire
// multiply-shift bounded draws), so seeded inputs are identical across
// standard libraries and identical to the oracle's generators.
#include <cstdint>
#include <vector>

#include "hetm_b200/capi.h"

namespace {

class SeqRng {
public:
    explicit SeqRng(uint64_t seed) : s_(seed == 0 ? 0x853c49e6748fea9bULL : seed) {}
    uint64_t next() {
        uint64_t z = s_ + 0x9e3779b97f4a7c15ULL;
        z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
        z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
        s_ = z ^ (z >> 31);
        return s_;
    }
    uint64_t below(uint64_t bound) { return (uint64_t)(((unsigned __int128)next() * bound) >> 64); }

private:
    uint64_t s_;
};

// Draws a value in [0, span) not among the first k of `taken` (rejection).
uint64_t fresh(SeqRng& r, uint64_t span, const uint64_t* taken, int k) {
    for (;;) {
        const uint64_t x = r.below(span);
        bool seen = false;
        for (int j = 0; j < k; ++j) seen = seen || taken[j] == x;
        if (!seen) return x;
    }
}

}  // namespace

extern "C" int hetm_gen_bank_batch(uint64_t seed, uint64_t n, uint64_t lo, uint64_t span, hetm_bank_tx* out) {
    if (!out && n) return HETM_ERR_INVALID_ARG;
    if (span < 4 || lo + span > (1ull << 32)) return HETM_ERR_INVALID_SIZE;
    SeqRng r(seed);
    for (uint64_t i = 0; i < n; ++i) {
        uint64_t picked[4];
        for (int k = 0; k < 4; ++k) picked[k] = fresh(r, span, picked, k);
        for (int k = 0; k < 4; ++k) out[i].acct[k] = (uint32_t)(lo + picked[k]);
        out[i].amount = r.below(100) + 1;
    }
    return HETM_OK;
}

extern "C" int hetm_gen_host_log(uint64_t seed, uint64_t n_tx, uint32_t writes_per_tx, uint32_t n_threads,
                                 uint64_t lo, uint64_t span, uint64_t ts_base, hetm_log_entry* out) {
    if (!out && n_tx) return HETM_ERR_INVALID_ARG;
    if (n_threads == 0 || writes_per_tx == 0 || writes_per_tx > 16 || span < writes_per_tx)
        return HETM_ERR_INVALID_SIZE;
    // Thread t's log holds transactions t, t+T, t+2T, ... and starts after the
    // logs of threads < t (WriteLog::allEntries order, write_log.hpp:74-82).
    std::vector<uint64_t> start(n_threads + 1, 0);
    for (uint32_t t = 0; t < n_threads; ++t) {
        const uint64_t txs = n_tx / n_threads + (t < n_tx % n_threads ? 1 : 0);
        start[t + 1] = start[t] + txs * writes_per_tx;
    }
    SeqRng r(seed);
    uint64_t picked[16];
    for (uint64_t i = 0; i < n_tx; ++i) {
        hetm_log_entry* e = out + start[i % n_threads] + (i / n_threads) * writes_per_tx;
        for (uint32_t k = 0; k < writes_per_tx; ++k) {
            picked[k] = fresh(r, span, picked, (int)k);
            e[k].addr = lo + picked[k];
            e[k].value = r.next();
            e[k].ts = ts_base + 1 + i;
        }
    }
    return HETM_OK;
}
