/*
 * hetm_oracle.c — CPU restatement of the Speculative HeTM GPU-side path.
 *
 * TEST INFRASTRUCTURE ONLY (see hetm_oracle.h).  Plain C11 + pthreads.
 * Parity status: RNG / bitmap geometry / log order pinned against the
 * reference headers (tests/golden/ref_vectors.json, oracle/ref_shim.cpp);
 * validate / replay / merge restate SPEC.md and are pinned by its examples
 * (tests/test_oracle.py) — the reference ships no implementation of them.
 */
#define _GNU_SOURCE
#include "hetm_oracle.h"

#include <math.h>
#include <pthread.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------ RNG --
 * det_rng.hpp:8-13 splitmix64; :21 zero-seed substitute; :23-26 next();
 * :29-33 below() as Lemire multiply-shift; :36 uniform() from the top 53 bits. */
uint64_t orc_splitmix64(uint64_t x) {
    x += 0x9e3779b97f4a7c15ULL;
    x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
    x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
    return x ^ (x >> 31);
}
void orc_rng_init(orc_rng* r, uint64_t seed) { r->state = seed ? seed : 0x853c49e6748fea9bULL; }
uint64_t orc_rng_next(orc_rng* r) { return r->state = orc_splitmix64(r->state); }
uint64_t orc_rng_below(orc_rng* r, uint64_t bound) {
    unsigned __int128 p = (unsigned __int128)orc_rng_next(r) * bound;
    return (uint64_t)(p >> 64);
}
double orc_rng_uniform(orc_rng* r) { return (double)(orc_rng_next(r) >> 11) * 0x1.0p-53; }

void orc_rng_fill_next(uint64_t seed, uint64_t n, uint64_t* out) {
    orc_rng r; orc_rng_init(&r, seed);
    for (uint64_t i = 0; i < n; ++i) out[i] = orc_rng_next(&r);
}
void orc_rng_fill_below(uint64_t seed, uint64_t bound, uint64_t n, uint64_t* out) {
    orc_rng r; orc_rng_init(&r, seed);
    for (uint64_t i = 0; i < n; ++i) out[i] = orc_rng_below(&r, bound);
}
void orc_rng_fill_uniform(uint64_t seed, uint64_t n, double* out) {
    orc_rng r; orc_rng_init(&r, seed);
    for (uint64_t i = 0; i < n; ++i) out[i] = orc_rng_uniform(&r);
}

/* -------------------------------------------------------------- bitmaps --
 * bitmap.hpp:96-97 bit count = ceil(region/gran); :99-100 gran pow2 and a
 * multiple of the 8-byte word; :104 bit covering a word = addr*8/gran;
 * :15-23 snapshot word layout bit b <-> words[b>>6] bit (b&63). */
uint64_t orc_bits_for_region(uint64_t region_bytes, uint64_t gran_bytes) {
    return (region_bytes + gran_bytes - 1) / gran_bytes;
}
int orc_valid_gran(uint64_t g) { return g != 0 && (g & (g - 1)) == 0 && g % 8 == 0; }
uint64_t orc_bit_of_word(uint64_t addr, uint64_t gran_bytes) { return addr * 8u / gran_bytes; }
void orc_bitmap_set(uint64_t* w, uint64_t bit) { w[bit >> 6] |= 1ULL << (bit & 63); }
int orc_bitmap_test(const uint64_t* w, uint64_t bit) { return (int)((w[bit >> 6] >> (bit & 63)) & 1u); }
uint64_t orc_popcount(const uint64_t* w, uint64_t n) {
    uint64_t c = 0;
    for (uint64_t i = 0; i < n; ++i) c += (uint64_t)__builtin_popcountll(w[i]);
    return c;
}

/* ------------------------------------------------------- validateChunk --
 * for each entry (a) RS bit covering addr set -> conflictFlag;
 * (b) apply mode, regardless of (a): if entry.ts > TS[addr].ts then
 * dev[addr] = value, TS[addr].ts = entry.ts.  Validate-only skips (b).
 * Single worker, entries in delivery order. */
int orc_validate_chunk(const orc_entry* e, uint64_t n, const uint64_t* rs, uint64_t gran,
                       uint64_t base, uint64_t* ts, uint64_t* dev, int apply) {
    int conflict = 0;
    for (uint64_t i = 0; i < n; ++i) {
        uint64_t a = e[i].addr - base;
        if (orc_bitmap_test(rs, orc_bit_of_word(a, gran))) conflict = 1;
        if (apply && e[i].ts > ts[a]) {
            dev[a] = e[i].value;
            ts[a] = e[i].ts;
        }
    }
    return conflict;
}

/* ---------------------------------------------------- bruteForceIntersect --
 * true iff any log entry's covering bit is set.  Written
 * independently of the validator: byte offsets and division,
 * bounds-checked against the bitmap size. */
int orc_brute_force_intersect(const orc_entry* e, uint64_t n, const uint64_t* rs, uint64_t rs_bits,
                              uint64_t gran, uint64_t base) {
    for (uint64_t i = 0; i < n; ++i) {
        uint64_t byte_off = (e[i].addr - base) * (uint64_t)sizeof(uint64_t);
        uint64_t bit = byte_off / gran;
        if (bit >= rs_bits) continue;
        uint64_t word = rs[bit / 64];
        if ((word >> (bit % 64)) & 1ULL) return 1;
    }
    return 0;
}

/* ----------------------------------------------------- sequentialReplay --
 * device txs in their serial order on one region.
 * Bitmap post-condition of executeBatch: reads set RS; writes
 * set WS *and* RS; written chunks set the ChunkMap. */
static void mark(uint64_t* bm, uint64_t a, uint64_t g) {
    if (bm) orc_bitmap_set(bm, orc_bit_of_word(a, g));
}

void orc_bank_replay(uint64_t* s, uint64_t base, const orc_bank_tx* tx, const uint64_t* order,
                     uint64_t n_order, uint64_t* rs, uint64_t* ws, uint64_t* ch, uint64_t gran,
                     uint64_t chunk) {
    for (uint64_t k = 0; k < n_order; ++k) {
        const orc_bank_tx* t = &tx[order[k]];
        uint64_t a[4];
        for (int j = 0; j < 4; ++j) {
            a[j] = (uint64_t)t->acct[j] - base;
            mark(rs, a[j], gran);
        }
        uint64_t v0 = s[a[0]], v1 = s[a[1]];
        s[a[0]] = v0 - t->amount;
        s[a[1]] = v1 + t->amount;
        for (int j = 0; j < 2; ++j) {
            mark(ws, a[j], gran);
            mark(ch, a[j], chunk);
        }
    }
}

void orc_rw_replay(uint64_t* s, uint64_t base, const orc_rw_tx* tx, const uint64_t* order,
                   uint64_t n_order, uint64_t* rs, uint64_t* ws, uint64_t* ch, uint64_t gran,
                   uint64_t chunk) {
    for (uint64_t k = 0; k < n_order; ++k) {
        const orc_rw_tx* t = &tx[order[k]];
        uint64_t sum = 0;
        for (uint32_t j = 0; j < t->nr && j < 4; ++j) {
            uint64_t a = t->r_addr[j] - base;
            sum += s[a];
            mark(rs, a, gran);
        }
        for (uint32_t j = 0; j < t->nw && j < 2; ++j) {
            uint64_t a = t->w_addr[j] - base;
            s[a] = s[a] + t->add[j] + sum; /* read-your-writes: sequential */
            mark(rs, a, gran);
            mark(ws, a, gran);
            mark(ch, a, chunk);
        }
    }
}

/* ------------------------------------------------ cache (configs[3]) --
 * MemcachedGPU-style set-associative cache (capi.h hetm_cache_*; PAPER.md:
 * 480-508): 8 ways x 8 words {key0,key1,value0..3,lru,
 * flags} per set; LRU stamp = serial position (device: ticket + 1). */
enum { C_WAYS = 8, C_WAYW = 8, C_SETW = 64, C_VAL = 2, C_LRU = 6, C_FLAGS = 7 };

uint64_t orc_cache_hash(uint64_t k0, uint64_t k1) {
    uint64_t z = k0 ^ (k1 * 0x9e3779b97f4a7c15ULL);
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
}
uint64_t orc_cache_set_of(uint64_t k0, uint64_t k1, uint64_t n_sets) {
    uint64_t half = n_sets / 2;
    return (k0 & 1) * half + (orc_cache_hash(k0, k1) & (half - 1));
}

static void cache_apply(uint64_t* s, uint64_t base, uint64_t cbase, uint64_t n_sets, const orc_cache_tx* t,
                        uint64_t stamp, orc_cache_result* out, uint64_t* rs, uint64_t* ws, uint64_t* ch,
                        uint64_t gran, uint64_t chunk, orc_entry* log, uint64_t* nlog, uint64_t ts) {
    const uint64_t s0 = cbase + orc_cache_set_of(t->key[0], t->key[1], n_sets) * C_SETW;
    int hit = C_WAYS, inv = C_WAYS, lru = 0;
    for (int w = 0; w < C_WAYS; ++w) {
        const uint64_t* way = s + s0 + (uint64_t)w * C_WAYW;
        if (hit == C_WAYS && (way[C_FLAGS] & 1) && way[0] == t->key[0] && way[1] == t->key[1]) hit = w;
        if (inv == C_WAYS && !(way[C_FLAGS] & 1)) inv = w;
        if (way[C_LRU] < s[s0 + (uint64_t)lru * C_WAYW + C_LRU]) lru = w;
        mark(rs, s0 + (uint64_t)w * C_WAYW + 0, gran);
        mark(rs, s0 + (uint64_t)w * C_WAYW + 1, gran);
        mark(rs, s0 + (uint64_t)w * C_WAYW + C_LRU, gran);
        mark(rs, s0 + (uint64_t)w * C_WAYW + C_FLAGS, gran);
    }
    int target;
    uint32_t status;
    if (t->op == 0) { target = hit; status = hit < C_WAYS ? 1 : 0; }
    else if (hit < C_WAYS) { target = hit; status = 2; }
    else if (inv < C_WAYS) { target = inv; status = 3; }
    else { target = lru; status = 4; }
    out->status = status;
    out->way = (uint32_t)target;
    for (int q = 0; q < 4; ++q) out->value[q] = 0;
    if (target == C_WAYS) return;
    uint64_t* way = s + s0 + (uint64_t)target * C_WAYW;
    const uint64_t wl = s0 + (uint64_t)target * C_WAYW;
    for (int q = 0; q < 4; ++q) {
        out->value[q] = t->op == 0 ? way[C_VAL + q] : t->value[q];
        mark(rs, wl + C_VAL + q, gran);
    }
    unsigned wmask = t->op == 0 ? (1u << C_LRU) : (status == 2 ? (0xfu << C_VAL) | (1u << C_LRU) : 0xffu);
    uint64_t nv[C_WAYW];
    for (int q = 0; q < C_WAYW; ++q) nv[q] = way[q];
    if (t->op == 1) {
        nv[0] = t->key[0];
        nv[1] = t->key[1];
        for (int q = 0; q < 4; ++q) nv[C_VAL + q] = t->value[q];
        nv[C_FLAGS] = 1;
    }
    nv[C_LRU] = stamp;
    for (int q = 0; q < C_WAYW; ++q) {
        if (!((wmask >> q) & 1u)) continue;
        way[q] = nv[q];
        mark(ws, wl + q, gran);
        mark(ch, wl + q, chunk);
        if (log) {
            log[*nlog].addr = base + wl + q;
            log[*nlog].value = nv[q];
            log[*nlog].ts = ts;
            ++*nlog;
        }
    }
}

void orc_cache_replay(uint64_t* s, uint64_t base, uint64_t cbase, uint64_t n_sets, const orc_cache_tx* tx,
                      const uint64_t* order, uint64_t n_order, const uint64_t* tickets, orc_cache_result* results,
                      uint64_t* rs, uint64_t* ws, uint64_t* ch, uint64_t gran, uint64_t chunk) {
    for (uint64_t k = 0; k < n_order; ++k) {
        const uint64_t i = order[k];
        cache_apply(s, base, cbase, n_sets, &tx[i], tickets[i] + 1, &results[i], rs, ws, ch, gran, chunk, NULL, NULL, 0);
    }
}

uint64_t orc_cache_host_run(uint64_t* s, uint64_t base, uint64_t cbase, uint64_t n_sets, const orc_cache_tx* tx,
                            uint64_t n, uint64_t ts_base, orc_cache_result* results, orc_entry* log) {
    uint64_t nlog = 0;
    for (uint64_t i = 0; i < n; ++i)
        cache_apply(s, base, cbase, n_sets, &tx[i], ts_base + 1 + i, &results[i], NULL, NULL, NULL, 8, 8, log, &nlog,
                    ts_base + 1 + i);
    return nlog;
}

static const uint64_t* g_sort_keys;
static int cmp_by_key(const void* x, const void* y) {
    uint64_t i = *(const uint64_t*)x, j = *(const uint64_t*)y;
    uint64_t a = g_sort_keys[i], b = g_sort_keys[j];
    if (a != b) return a < b ? -1 : 1;
    return i < j ? -1 : (i > j);
}
uint64_t orc_order_by_ticket(const uint64_t* tickets, uint64_t n, uint64_t* order) {
    uint64_t m = 0;
    for (uint64_t i = 0; i < n; ++i)
        if (tickets[i] != UINT64_MAX) order[m++] = i;
    g_sort_keys = tickets;
    qsort(order, m, sizeof(uint64_t), cmp_by_key);
    return m;
}

/* ------------------------------------------------------------ coalescing --
 * adjacent dirty chunks become one transfer descriptor;
 * 2 adjacent 16 KiB chunks -> one record of 32768 bytes.
 * The last chunk is clipped to the region end. */
uint64_t orc_coalesce_chunks(const uint64_t* cw, uint64_t n_chunks, uint64_t chunk, uint64_t region,
                             orc_range* out, uint64_t max_out) {
    uint64_t m = 0, c = 0;
    while (c < n_chunks) {
        if (!orc_bitmap_test(cw, c)) { ++c; continue; }
        uint64_t start = c;
        while (c < n_chunks && orc_bitmap_test(cw, c)) ++c;
        uint64_t lo = start * chunk, hi = c * chunk;
        if (hi > region) hi = region;
        if (m < max_out) { out[m].offset_bytes = lo; out[m].bytes = hi - lo; }
        ++m;
    }
    return m;
}

/* -------------------------------------------------- ts-ordered log apply --
 * SPEC.md:375 optimized rollback: the round's full host log applied in ts
 * order (ties — entries of one transaction — touch distinct words). */
static const orc_entry* g_sort_log;
static int cmp_log(const void* x, const void* y) {
    uint64_t i = *(const uint64_t*)x, j = *(const uint64_t*)y;
    uint64_t a = g_sort_log[i].ts, b = g_sort_log[j].ts;
    if (a != b) return a < b ? -1 : 1;
    return i < j ? -1 : (i > j);
}
void orc_apply_log_ts_order(uint64_t* region, uint64_t base, const orc_entry* e, uint64_t n) {
    uint64_t* idx = (uint64_t*)malloc(sizeof(uint64_t) * (n ? n : 1));
    for (uint64_t i = 0; i < n; ++i) idx[i] = i;
    g_sort_log = e;
    qsort(idx, n, sizeof(uint64_t), cmp_log);
    for (uint64_t k = 0; k < n; ++k) region[e[idx[k]].addr - base] = e[idx[k]].value;
    free(idx);
}

/* ---------------------------------------------------------- generators -- */
/* Zipf(alpha) ranks 1..n by rejection-inversion (W. Hormann, G. Derflinger,
 * "Rejection-inversion to generate variates from monotone discrete
 * distributions", ACM TOMACS 6(3), 1996), one DetRng uniform() per trial
 * (det_rng.hpp:36).  The reference pins only the sampler's law (SPEC.md:620:
 * top-10 rank frequencies within 5% of the analytic law at alpha 0.5). */
typedef struct { double s, n, hx1, hxn, sdiv; } orc_zipf;
static double zf_h1(double x) { return fabs(x) > 1e-8 ? log1p(x) / x : 1.0 - x * (0.5 - x * (1.0 / 3.0 - 0.25 * x)); }
static double zf_h2(double x) { return fabs(x) > 1e-8 ? expm1(x) / x : 1.0 + x * 0.5 * (1.0 + x * (1.0 / 3.0) * (1.0 + 0.25 * x)); }
static double zf_hint(const orc_zipf* z, double x) { const double lx = log(x); return zf_h2((1.0 - z->s) * lx) * lx; }
static double zf_h(const orc_zipf* z, double x) { return exp(-z->s * log(x)); }
static double zf_hinv(const orc_zipf* z, double x) {
    double t = x * (1.0 - z->s);
    if (t < -1.0) t = -1.0;
    return exp(zf_h1(t) * x);
}
static void zf_init(orc_zipf* z, double alpha, uint64_t n) {
    z->s = alpha;
    z->n = (double)n;
    z->hx1 = zf_hint(z, 1.5) - 1.0;
    z->hxn = zf_hint(z, z->n + 0.5);
    z->sdiv = 2.0 - zf_hinv(z, zf_hint(z, 2.5) - zf_h(z, 2.0));
}
static uint64_t zf_sample(const orc_zipf* z, orc_rng* r) {
    for (;;) {
        const double u = z->hxn + orc_rng_uniform(r) * (z->hx1 - z->hxn);
        const double x = zf_hinv(z, u);
        double kd = floor(x + 0.5);
        if (kd < 1.0) kd = 1.0;
        else if (kd > z->n) kd = z->n;
        if (kd - x <= z->sdiv || u >= zf_hint(z, kd + 0.5) - zf_h(z, kd)) return (uint64_t)kd;
    }
}

void orc_zipf_fill(uint64_t seed, uint64_t n, uint64_t span, double alpha, uint64_t* out) {
    orc_rng r; orc_rng_init(&r, seed);
    orc_zipf z; zf_init(&z, alpha, span);
    for (uint64_t i = 0; i < n; ++i) out[i] = zf_sample(&z, &r);
}

/* offset in [0, span): uniform below(span) (alpha == 0) or zipf rank - 1 */
static uint64_t draw_offset(orc_rng* r, uint64_t span, const orc_zipf* z) {
    return z ? zf_sample(z, r) - 1 : orc_rng_below(r, span);
}

static uint64_t draw_distinct(orc_rng* r, uint64_t span, const orc_zipf* z, const uint64_t* prev, int nprev) {
    for (;;) {
        uint64_t a = draw_offset(r, span, z);
        int dup = 0;
        for (int k = 0; k < nprev; ++k) dup |= (prev[k] == a);
        if (!dup) return a;
    }
}

void orc_gen_bank_batch_zipf(uint64_t seed, uint64_t n, uint64_t lo, uint64_t span, double alpha, orc_bank_tx* out) {
    orc_rng r; orc_rng_init(&r, seed);
    orc_zipf z; zf_init(&z, alpha > 0 ? alpha : 1.0, span);
    const orc_zipf* zp = alpha > 0 ? &z : NULL;
    for (uint64_t i = 0; i < n; ++i) {
        uint64_t a[4];
        for (int k = 0; k < 4; ++k) a[k] = draw_distinct(&r, span, zp, a, k);
        for (int k = 0; k < 4; ++k) out[i].acct[k] = (uint32_t)(lo + a[k]);
        out[i].amount = orc_rng_below(&r, 100) + 1;
    }
}

void orc_gen_bank_batch(uint64_t seed, uint64_t n, uint64_t lo, uint64_t span, orc_bank_tx* out) {
    orc_gen_bank_batch_zipf(seed, n, lo, span, 0.0, out);
}

void orc_gen_host_log_zipf(uint64_t seed, uint64_t n_tx, uint32_t wpt, uint32_t T, uint64_t lo, uint64_t span,
                           uint64_t ts_base, double alpha, orc_entry* out) {
    orc_rng r; orc_rng_init(&r, seed);
    orc_zipf z; zf_init(&z, alpha > 0 ? alpha : 1.0, span);
    const orc_zipf* zp = alpha > 0 ? &z : NULL;
    /* thread t receives txs t, t+T, ...; its log starts after threads < t */
    uint64_t* off = (uint64_t*)calloc(T + 1, sizeof(uint64_t));
    for (uint32_t t = 0; t < T; ++t) {
        uint64_t cnt = n_tx / T + (t < n_tx % T ? 1 : 0);
        off[t + 1] = off[t] + cnt * wpt;
    }
    uint64_t prev[16];
    for (uint64_t i = 0; i < n_tx; ++i) {
        uint32_t t = (uint32_t)(i % T);
        uint64_t pos = off[t] + (i / T) * wpt;
        for (uint32_t k = 0; k < wpt; ++k) {
            uint64_t a = draw_distinct(&r, span, zp, prev, (int)(k < 16 ? k : 16));
            if (k < 16) prev[k] = a;
            out[pos + k].addr = lo + a;
            out[pos + k].value = orc_rng_next(&r);
            out[pos + k].ts = ts_base + 1 + i;
        }
    }
    free(off);
}

void orc_gen_host_log(uint64_t seed, uint64_t n_tx, uint32_t wpt, uint32_t T, uint64_t lo,
                      uint64_t span, uint64_t ts_base, orc_entry* out) {
    orc_gen_host_log_zipf(seed, n_tx, wpt, T, lo, span, ts_base, 0.0, out);
}

void orc_gen_cache_batch(uint64_t seed, uint64_t n, uint64_t key_space, double alpha, uint32_t get_permille,
                         int32_t part, uint32_t steal_permille, orc_cache_tx* out) {
    orc_rng r; orc_rng_init(&r, seed);
    orc_zipf z; zf_init(&z, alpha > 0 ? alpha : 1.0, key_space);
    for (uint64_t i = 0; i < n; ++i) {
        const uint64_t rank = alpha > 0 ? zf_sample(&z, &r) : orc_rng_below(&r, key_space) + 1;
        uint64_t p = (uint64_t)part;
        if (part < 0) p = orc_rng_below(&r, 1000) < steal_permille ? 0 : 1;
        out[i].op = orc_rng_below(&r, 1000) < get_permille ? 0 : 1;
        out[i].reserved = 0;
        out[i].key[0] = (orc_splitmix64(rank) & ~1ULL) | p;
        out[i].key[1] = rank;
        for (int q = 0; q < 4; ++q) out[i].value[q] = out[i].op == 1 ? orc_rng_next(&r) : 0;
    }
}

/* ------------------------------------------------------- CPU baselines -- */
#define LOCKBIT (1ULL << 63)

static inline uint64_t lk_index(uint64_t a, uint64_t lock_entries) {
    return (a * 0x9E3779B97F4A7C15ULL) & (lock_entries - 1);
}

typedef struct {
    uint64_t* s; uint64_t base; const orc_bank_tx* tx; uint64_t lo, hi;
    uint64_t* locks; uint64_t nlocks; uint64_t* ticket; uint64_t* tickets_out;
    uint64_t* rs; uint64_t* ws; uint64_t* ch; uint64_t gran, chunk;
    uint64_t committed;
} bank_job;

static void atomic_or(uint64_t* w, uint64_t bit) {
    if (w) __atomic_fetch_or(&w[bit >> 6], 1ULL << (bit & 63), __ATOMIC_RELAXED);
}

/* TL2-style commit-time locking: versioned lock per
 * (hashed) word; lock write set in address order, take the commit ticket,
 * validate the read set, write back, release with version = ticket. */
static void* bank_worker(void* p) {
    bank_job* j = (bank_job*)p;
    for (uint64_t i = j->lo; i < j->hi; ++i) {
        const orc_bank_tx* t = &j->tx[i];
        uint64_t a[4], l[4], ver[4], v[4];
        for (int k = 0; k < 4; ++k) { a[k] = (uint64_t)t->acct[k] - j->base; l[k] = lk_index(a[k], j->nlocks); }
        for (;;) {
            int ok = 1;
            for (int k = 0; k < 4 && ok; ++k) {
                uint64_t x = __atomic_load_n(&j->locks[l[k]], __ATOMIC_ACQUIRE);
                if (x & LOCKBIT) { ok = 0; break; }
                v[k] = __atomic_load_n(&j->s[a[k]], __ATOMIC_ACQUIRE);
                uint64_t y = __atomic_load_n(&j->locks[l[k]], __ATOMIC_ACQUIRE);
                if (y != x) ok = 0;
                ver[k] = x;
            }
            if (!ok) continue;
            /* write-lock entries l[0], l[1] in index order, deduplicated */
            uint64_t w0 = l[0] < l[1] ? l[0] : l[1], w1 = l[0] < l[1] ? l[1] : l[0];
            uint64_t wl[2] = {w0, w1};
            int nwl = (w0 == w1) ? 1 : 2, held = 0;
            for (int k = 0; k < nwl; ++k) {
                uint64_t expect = (wl[k] == l[0]) ? ver[0] : ver[1];
                if (!__atomic_compare_exchange_n(&j->locks[wl[k]], &expect, expect | LOCKBIT, 0,
                                                 __ATOMIC_ACQ_REL, __ATOMIC_RELAXED))
                    break;
                ++held;
            }
            if (held < nwl) {
                for (int k = 0; k < held; ++k)
                    __atomic_fetch_and(&j->locks[wl[k]], ~LOCKBIT, __ATOMIC_RELEASE);
                continue;
            }
            uint64_t tk = __atomic_fetch_add(j->ticket, 1, __ATOMIC_ACQ_REL);
            for (int k = 2; k < 4 && ok; ++k) {
                if (l[k] == w0 || l[k] == w1) continue;
                if (__atomic_load_n(&j->locks[l[k]], __ATOMIC_ACQUIRE) != ver[k]) ok = 0;
            }
            if (!ok) {
                for (int k = 0; k < nwl; ++k)
                    __atomic_fetch_and(&j->locks[wl[k]], ~LOCKBIT, __ATOMIC_RELEASE);
                continue;
            }
            __atomic_store_n(&j->s[a[0]], v[0] - t->amount, __ATOMIC_RELAXED);
            __atomic_store_n(&j->s[a[1]], v[1] + t->amount, __ATOMIC_RELAXED);
            for (int k = 0; k < nwl; ++k)
                __atomic_store_n(&j->locks[wl[k]], (tk + 1) & ~LOCKBIT, __ATOMIC_RELEASE);
            if (j->tickets_out) j->tickets_out[i] = tk;
            for (int k = 0; k < 4; ++k) atomic_or(j->rs, orc_bit_of_word(a[k], j->gran));
            for (int k = 0; k < 2; ++k) {
                atomic_or(j->ws, orc_bit_of_word(a[k], j->gran));
                atomic_or(j->ch, orc_bit_of_word(a[k], j->chunk));
            }
            j->committed++;
            break;
        }
    }
    return NULL;
}

uint64_t orc_mt_bank_batch(uint64_t* s, uint64_t base, uint64_t size_words, const orc_bank_tx* tx,
                           uint64_t n, int T, uint64_t nlocks, uint64_t* tickets_out, uint64_t* rs,
                           uint64_t* ws, uint64_t* ch, uint64_t gran, uint64_t chunk) {
    (void)size_words;
    if (T < 1) T = 1;
    uint64_t* locks = (uint64_t*)calloc(nlocks, sizeof(uint64_t));
    uint64_t ticket = 0;
    pthread_t* th = (pthread_t*)calloc((size_t)T, sizeof(pthread_t));
    bank_job* jobs = (bank_job*)calloc((size_t)T, sizeof(bank_job));
    for (int t = 0; t < T; ++t) {
        bank_job* j = &jobs[t];
        j->s = s; j->base = base; j->tx = tx; j->lo = n * (uint64_t)t / (uint64_t)T;
        j->hi = n * (uint64_t)(t + 1) / (uint64_t)T; j->locks = locks; j->nlocks = nlocks;
        j->ticket = &ticket; j->tickets_out = tickets_out; j->rs = rs; j->ws = ws; j->ch = ch;
        j->gran = gran; j->chunk = chunk;
        pthread_create(&th[t], NULL, bank_worker, j);
    }
    uint64_t c = 0;
    for (int t = 0; t < T; ++t) { pthread_join(th[t], NULL); c += jobs[t].committed; }
    free(th); free(jobs); free(locks);
    return c;
}

typedef struct {
    const orc_entry* e; uint64_t lo, hi; const uint64_t* rs; uint64_t gran, base;
    uint64_t* ts; uint64_t* dev; int apply; int conflict;
} val_job;

/* PAPER.md:330 / SPEC.md:348: take the TS lock bit, compare, apply, release. */
static void* val_worker(void* p) {
    val_job* j = (val_job*)p;
    int c = 0;
    for (uint64_t i = j->lo; i < j->hi; ++i) {
        uint64_t a = j->e[i].addr - j->base;
        c |= orc_bitmap_test(j->rs, orc_bit_of_word(a, j->gran));
        if (!j->apply) continue;
        uint64_t ts = j->e[i].ts;
        uint64_t cur = __atomic_load_n(&j->ts[a], __ATOMIC_RELAXED);
        for (;;) {
            if (!(cur & LOCKBIT) && cur >= ts) break; /* not fresher: skip */
            if (cur & LOCKBIT) { cur = __atomic_load_n(&j->ts[a], __ATOMIC_RELAXED); continue; }
            if (__atomic_compare_exchange_n(&j->ts[a], &cur, cur | LOCKBIT, 0, __ATOMIC_ACQUIRE,
                                            __ATOMIC_RELAXED)) {
                __atomic_store_n(&j->dev[a], j->e[i].value, __ATOMIC_RELAXED);
                __atomic_store_n(&j->ts[a], ts, __ATOMIC_RELEASE);
                break;
            }
        }
    }
    j->conflict = c;
    return NULL;
}

int orc_mt_validate_apply(const orc_entry* e, uint64_t n, const uint64_t* rs, uint64_t gran,
                          uint64_t base, uint64_t* ts, uint64_t* dev, int T, int apply) {
    if (T < 1) T = 1;
    pthread_t* th = (pthread_t*)calloc((size_t)T, sizeof(pthread_t));
    val_job* jobs = (val_job*)calloc((size_t)T, sizeof(val_job));
    for (int t = 0; t < T; ++t) {
        val_job* j = &jobs[t];
        j->e = e; j->lo = n * (uint64_t)t / (uint64_t)T; j->hi = n * (uint64_t)(t + 1) / (uint64_t)T;
        j->rs = rs; j->gran = gran; j->base = base; j->ts = ts; j->dev = dev; j->apply = apply;
        pthread_create(&th[t], NULL, val_worker, j);
    }
    int c = 0;
    for (int t = 0; t < T; ++t) { pthread_join(th[t], NULL); c |= jobs[t].conflict; }
    free(th); free(jobs);
    return c;
}
