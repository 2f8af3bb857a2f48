// gen.cpp — seeded host-side input generators (bank batches, host write logs).
//
// Deterministic generator per det_rng.hpp:8-42 (splitmix64 state walk, Lemire
// multiply-shift bounded draws), so seeded inputs are identical across
// standard libraries and identical to the oracle's generators.
#include <cmath>
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
    double uniform() { return (double)(next() >> 11) * 0x1.0p-53; }  // det_rng.hpp:36

private:
    uint64_t s_;
};

// Zipf(alpha) over ranks 1..n by rejection-inversion (Hormann & Derflinger,
// ACM TOMACS 6(3), 1996): O(1) per draw for any n, one uniform() per trial.
class Zipf {
public:
    Zipf(double alpha, uint64_t n) : s_(alpha), n_((double)n) {
        hx1_ = hint(1.5) - 1.0;
        hxn_ = hint(n_ + 0.5);
        sdiv_ = 2.0 - hinv(hint(2.5) - h(2.0));
    }
    uint64_t rank(SeqRng& r) const {
        for (;;) {
            const double u = hxn_ + r.uniform() * (hx1_ - hxn_);
            const double x = hinv(u);
            const double k = std::fmin(std::fmax(std::floor(x + 0.5), 1.0), n_);
            if (k - x <= sdiv_ || u >= hint(k + 0.5) - h(k)) return (uint64_t)k;
        }
    }

private:
    static double log1p_over(double x) { return std::fabs(x) > 1e-8 ? std::log1p(x) / x : 1.0 - x * (0.5 - x * (1.0 / 3.0 - 0.25 * x)); }
    static double expm1_over(double x) {
        return std::fabs(x) > 1e-8 ? std::expm1(x) / x : 1.0 + x * 0.5 * (1.0 + x * (1.0 / 3.0) * (1.0 + 0.25 * x));
    }
    double hint(double x) const {
        const double lx = std::log(x);
        return expm1_over((1.0 - s_) * lx) * lx;
    }
    double h(double x) const { return std::exp(-s_ * std::log(x)); }
    double hinv(double x) const { return std::exp(log1p_over(std::fmax(x * (1.0 - s_), -1.0)) * x); }
    double s_, n_, hx1_, hxn_, sdiv_;
};

// Offsets in [0, span): uniform below(span), or zipf rank - 1 (rank 1 hottest).
struct Sampler {
    uint64_t span;
    const Zipf* zipf;
    uint64_t draw(SeqRng& r) const { return zipf ? zipf->rank(r) - 1 : r.below(span); }
    // a value not among the first k of `taken` (rejection)
    uint64_t fresh(SeqRng& r, const uint64_t* taken, int k) const {
        for (;;) {
            const uint64_t x = draw(r);
            bool seen = false;
            for (int j = 0; j < k; ++j) seen = seen || taken[j] == x;
            if (!seen) return x;
        }
    }
};

int bank_batch(uint64_t seed, uint64_t n, uint64_t lo, uint64_t span, double alpha, hetm_bank_tx* out) {
    if (!out && n) return HETM_ERR_INVALID_ARG;
    if (span < 4 || lo + span > (1ull << 32) || !(alpha >= 0.0)) return HETM_ERR_INVALID_SIZE;
    const Zipf z(alpha > 0 ? alpha : 1.0, span);
    const Sampler smp{span, alpha > 0 ? &z : nullptr};
    SeqRng r(seed);
    for (uint64_t i = 0; i < n; ++i) {
        uint64_t picked[4];
        for (int k = 0; k < 4; ++k) picked[k] = smp.fresh(r, picked, k);
        for (int k = 0; k < 4; ++k) out[i].acct[k] = (uint32_t)(lo + picked[k]);
        out[i].amount = r.below(100) + 1;
    }
    return HETM_OK;
}

int host_log(uint64_t seed, uint64_t n_tx, uint32_t writes_per_tx, uint32_t n_threads, uint64_t lo, uint64_t span,
             uint64_t ts_base, double alpha, hetm_log_entry* out) {
    if (!out && n_tx) return HETM_ERR_INVALID_ARG;
    if (n_threads == 0 || writes_per_tx == 0 || writes_per_tx > 16 || span < writes_per_tx || !(alpha >= 0.0))
        return HETM_ERR_INVALID_SIZE;
    const Zipf z(alpha > 0 ? alpha : 1.0, span);
    const Sampler smp{span, alpha > 0 ? &z : nullptr};
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
            picked[k] = smp.fresh(r, picked, (int)k);
            e[k].addr = lo + picked[k];
            e[k].value = r.next();
            e[k].ts = ts_base + 1 + i;
        }
    }
    return HETM_OK;
}

uint64_t mix64(uint64_t x) {  // splitmix64 output function (det_rng.hpp:8-13)
    uint64_t z = x + 0x9e3779b97f4a7c15ULL;
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
}

}  // namespace

extern "C" int hetm_gen_cache_batch(uint64_t seed, uint64_t n, uint64_t key_space, double alpha, uint32_t get_permille,
                                    int32_t part, uint32_t steal_permille, hetm_cache_tx* out) {
    if (!out && n) return HETM_ERR_INVALID_ARG;
    if (key_space < 1 || get_permille > 1000 || steal_permille > 1000 || part > 1 || !(alpha >= 0.0))
        return HETM_ERR_INVALID_SIZE;
    const Zipf z(alpha > 0 ? alpha : 1.0, key_space);
    SeqRng r(seed);
    for (uint64_t i = 0; i < n; ++i) {
        const uint64_t rank = alpha > 0 ? z.rank(r) : r.below(key_space) + 1;
        uint64_t p = (uint64_t)part;
        if (part < 0) p = r.below(1000) < steal_permille ? 0 : 1;
        hetm_cache_tx& t = out[i];
        t.op = r.below(1000) < get_permille ? HETM_CACHE_GET : HETM_CACHE_SET;
        t.reserved = 0;
        t.key[0] = (mix64(rank) & ~1ull) | p;
        t.key[1] = rank;
        for (int q = 0; q < 4; ++q) t.value[q] = t.op == HETM_CACHE_SET ? r.next() : 0;
    }
    return HETM_OK;
}

extern "C" int hetm_gen_bank_batch(uint64_t seed, uint64_t n, uint64_t lo, uint64_t span, hetm_bank_tx* out) {
    return bank_batch(seed, n, lo, span, 0.0, out);
}

extern "C" int hetm_gen_bank_batch_zipf(uint64_t seed, uint64_t n, uint64_t lo, uint64_t span, double alpha,
                                        hetm_bank_tx* out) {
    return bank_batch(seed, n, lo, span, alpha, out);
}

extern "C" int hetm_gen_host_log(uint64_t seed, uint64_t n_tx, uint32_t writes_per_tx, uint32_t n_threads,
                                 uint64_t lo, uint64_t span, uint64_t ts_base, hetm_log_entry* out) {
    return host_log(seed, n_tx, writes_per_tx, n_threads, lo, span, ts_base, 0.0, out);
}

extern "C" int hetm_gen_host_log_zipf(uint64_t seed, uint64_t n_tx, uint32_t writes_per_tx, uint32_t n_threads,
                                      uint64_t lo, uint64_t span, uint64_t ts_base, double alpha,
                                      hetm_log_entry* out) {
    return host_log(seed, n_tx, writes_per_tx, n_threads, lo, span, ts_base, alpha, out);
}
