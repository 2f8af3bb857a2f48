/*
 * checker.c — P1 / P2-dagger consistency checker over execution traces
 * (the `checker` module).  TEST INFRASTRUCTURE ONLY (see
 * hetm_oracle.h); checking is offline and single-threaded.
 *
 * Trace: hetm_trace_event records (include/hetm_b200/capi.h, mirrored here as
 * orc_trace_event).  A transaction is the set of events with one tx id:
 * BEGIN, READ(addr, value) / WRITE(addr, value) in program order,
 * SPEC_COMMIT(ts | ticket), then FINAL_COMMIT or ABORT(round); an attempt
 * that aborted before committing has ABORT(conflict) and is ignored.
 *
 * checkP1 (§3 P1): the finally committed
 * transactions must be explained by ONE serial order respecting real-time
 * order; the candidate is the engine's claimed order — per round, host
 * transactions by commit ts (a read-only one right after the update that
 * produced its snapshot), then device transactions by commit ticket
 * (PAPER.md Appendix: CPU serializes before GPU).  Every read must return the
 * latest preceding write in that order (own writes first); the first
 * inconsistent read is the witness.  Real time: a host transaction that began
 * after another's commit must follow it; device tickets must follow batch
 * order.
 *
 * checkP2dagger: every speculatively committed transaction
 * of an aborted side must be explained by the finally committed transactions
 * plus the speculative ones of its own device: its side's claimed local order
 * replayed on the round-start state (or on the round-start state plus the
 * other side's committed transactions of the round), exhaustively permuted
 * when the speculative set has <= 6 transactions.
 */
#include <stdlib.h>
#include <string.h>

#include "hetm_oracle.h"

enum { EV_BEGIN = 0, EV_READ = 1, EV_WRITE = 2, EV_SPEC = 3, EV_FINAL = 4, EV_ABORT = 5, EV_ROUND = 6 };
enum { ABORT_CONFLICT = 1, ABORT_ROUND = 2 };

typedef struct {
    uint64_t id, key, begin_seq, spec_seq;
    uint32_t round;
    uint8_t device, has_spec, has_final, has_abort, has_abort_round, read_only, has_begin;
    uint64_t op_lo, op_n; /* READ/WRITE events, program order, in ops[] */
} txrec;

static int cmp_tx_seq(const void* a, const void* b) {
    const orc_trace_event* x = *(const orc_trace_event* const*)a;
    const orc_trace_event* y = *(const orc_trace_event* const*)b;
    if (x->tx != y->tx) return x->tx < y->tx ? -1 : 1;
    return x->seq < y->seq ? -1 : x->seq > y->seq;
}

/* claimed order inside a round: host (key = 2 ts + read_only) before device (key = ticket) */
static int cmp_claimed(const void* a, const void* b) {
    const txrec* x = *(const txrec* const*)a;
    const txrec* y = *(const txrec* const*)b;
    if (x->round != y->round) return x->round < y->round ? -1 : 1;
    if (x->device != y->device) return x->device < y->device ? -1 : 1;
    if (x->key != y->key) return x->key < y->key ? -1 : 1;
    return x->id < y->id ? -1 : x->id > y->id;
}

typedef struct {
    uint64_t seq;
    txrec* t;
    int is_commit;
} mark;
static int cmp_mark(const void* a, const void* b) {
    const mark* x = a;
    const mark* y = b;
    return x->seq < y->seq ? -1 : x->seq > y->seq;
}

/* ---- a small open-addressing overlay {addr -> value} over a base state */
typedef struct {
    uint64_t *k, *v;
    uint8_t* used;
    uint64_t mask;
} overlay;

static int ov_init(overlay* o, uint64_t n) {
    uint64_t cap = 16;
    while (cap < 2 * n + 16) cap <<= 1;
    o->k = calloc(cap, 8);
    o->v = calloc(cap, 8);
    o->used = calloc(cap, 1);
    o->mask = cap - 1;
    return o->k && o->v && o->used;
}
static void ov_free(overlay* o) {
    free(o->k);
    free(o->v);
    free(o->used);
}
static void ov_clear(overlay* o) { memset(o->used, 0, o->mask + 1); }
static uint64_t* ov_find(overlay* o, uint64_t a, int insert) {
    uint64_t h = (a * 0x9e3779b97f4a7c15ull) & o->mask;
    while (o->used[h]) {
        if (o->k[h] == a) return &o->v[h];
        h = (h + 1) & o->mask;
    }
    if (!insert) return NULL;
    o->used[h] = 1;
    o->k[h] = a;
    return &o->v[h];
}

typedef struct {
    const orc_trace_event* const* ops;
    const uint64_t* base; /* committed state */
    uint64_t words;
    overlay* ov;          /* NULL: write straight into `state` */
    uint64_t* state;
    orc_check_result* res;
    int check_reads;      /* 0: publish the writes only */
} replay_ctx;

/* Replays one transaction: checks its reads, then publishes its writes.
 * Returns 0 or 1 (inconsistent read / bad address, witness in res). */
static int replay_tx(replay_ctx* c, const txrec* t) {
    uint64_t wa[16], wv[16];
    int nw = 0;
    for (uint64_t k = 0; k < t->op_n; ++k) {
        const orc_trace_event* e = c->ops[t->op_lo + k];
        if (e->addr >= c->words) {
            c->res->verdict = ORC_CHECK_FAIL;
            c->res->reason = ORC_REASON_BAD_ADDR;
            c->res->tx = t->id;
            c->res->addr = e->addr;
            c->res->round = t->round;
            return 1;
        }
        int own = -1;
        for (int j = nw - 1; j >= 0 && own < 0; --j)
            if (wa[j] == e->addr) own = j;
        if (e->kind == EV_READ) {
            uint64_t cur;
            if (own >= 0) cur = wv[own];
            else if (c->ov) {
                const uint64_t* p = ov_find(c->ov, e->addr, 0);
                cur = p ? *p : c->base[e->addr];
            } else cur = c->state[e->addr];
            if (!c->check_reads) continue;
            c->res->checked_reads++;
            if (cur != e->value) {
                c->res->verdict = ORC_CHECK_FAIL;
                c->res->reason = ORC_REASON_READ;
                c->res->tx = t->id;
                c->res->addr = e->addr;
                c->res->expected = cur;
                c->res->got = e->value;
                c->res->round = t->round;
                return 1;
            }
        } else {
            if (own >= 0) wv[own] = e->value;
            else if (nw < 16) {
                wa[nw] = e->addr;
                wv[nw++] = e->value;
            }
        }
    }
    for (int j = 0; j < nw; ++j) {
        if (c->ov) *ov_find(c->ov, wa[j], 1) = wv[j];
        else c->state[wa[j]] = wv[j];
    }
    c->res->checked_txs += c->check_reads;
    return 0;
}

static int next_perm(txrec** a, int n) { /* lexicographic by pointer value */
    int i = n - 2;
    while (i >= 0 && a[i] >= a[i + 1]) --i;
    if (i < 0) return 0;
    int j = n - 1;
    while (a[j] <= a[i]) --j;
    txrec* t = a[i];
    a[i] = a[j];
    a[j] = t;
    for (int l = i + 1, r = n - 1; l < r; ++l, --r) {
        t = a[l];
        a[l] = a[r];
        a[r] = t;
    }
    return 1;
}
static int cmp_ptr(const void* a, const void* b) {
    const void* x = *(const void* const*)a;
    const void* y = *(const void* const*)b;
    return x < y ? -1 : x > y;
}

/* P2-dagger for one aborted side of one round: spec[0..ns) in claimed order;
 * extra[0..nx) = the other side's committed transactions of the round. */
static int check_spec_set(replay_ctx* c, txrec** spec, uint64_t ns, txrec** extra, uint64_t nx) {
    orc_check_result first = *c->res;
    for (int with_extra = 0; with_extra < 2; ++with_extra) {
        if (with_extra && !nx) break;
        txrec* perm[6];
        const int exhaustive = ns <= 6;
        if (exhaustive) {
            for (uint64_t i = 0; i < ns; ++i) perm[i] = spec[i];
        }
        int first_try = 1;
        for (;;) {
            ov_clear(c->ov);
            orc_check_result r = *c->res;
            replay_ctx cc = *c;
            cc.res = &r;
            int bad = 0;
            if (with_extra) { /* the other side's committed transactions first (checked by P1: writes only) */
                cc.check_reads = 0;
                for (uint64_t i = 0; i < nx; ++i) (void)replay_tx(&cc, extra[i]);
                cc.check_reads = 1;
            }
            for (uint64_t i = 0; i < ns && !bad; ++i) bad = replay_tx(&cc, exhaustive && !first_try ? perm[i] : spec[i]);
            if (!bad) {
                c->res->checked_txs = r.checked_txs;
                c->res->checked_reads = r.checked_reads;
                return 0;
            }
            if (first_try && !with_extra) first = r;
            if (!exhaustive) break;
            if (first_try) {
                qsort(perm, ns, sizeof perm[0], cmp_ptr);
                first_try = 0;
            } else if (!next_perm(perm, (int)ns)) break;
        }
    }
    *c->res = first;
    c->res->verdict = ORC_CHECK_FAIL;
    return 1;
}

static int check_trace(const orc_trace_event* ev, uint64_t n, const uint64_t* init, uint64_t words, int want_p2,
                       orc_check_result* res) {
    memset(res, 0, sizeof *res);
    res->verdict = ORC_CHECK_PASS;
    if (n == 0) return ORC_CHECK_PASS;  /* empty trace -> pass */
    const orc_trace_event** srt = malloc(n * sizeof *srt);
    const orc_trace_event** ops = malloc(n * sizeof *ops);
    txrec* txs = calloc(n, sizeof *txs);
    txrec** order = malloc(n * sizeof *order);
    uint64_t* state = malloc(words * 8);
    if (!srt || !ops || !txs || !order || !state) {
        free(srt), free(ops), free(txs), free(order), free(state);
        res->verdict = ORC_CHECK_INCOMPLETE;
        return res->verdict;
    }
    uint64_t m = 0;
    for (uint64_t i = 0; i < n; ++i)
        if (ev[i].kind != EV_ROUND) srt[m++] = &ev[i];
    qsort(srt, m, sizeof *srt, cmp_tx_seq);
    uint64_t nt = 0, nops = 0;
    for (uint64_t i = 0; i < m;) {
        txrec* t = &txs[nt++];
        t->id = srt[i]->tx;
        t->device = srt[i]->device;
        t->op_lo = nops;
        for (; i < m && srt[i]->tx == t->id; ++i) {
            const orc_trace_event* e = srt[i];
            switch (e->kind) {
                case EV_BEGIN: t->has_begin = 1; t->begin_seq = e->seq; t->round = e->round; break;
                case EV_READ: case EV_WRITE: ops[nops++] = e; break;
                case EV_SPEC: t->has_spec = 1; t->spec_seq = e->seq; t->key = e->value; t->round = e->round; break;
                case EV_FINAL: t->has_final = 1; break;
                case EV_ABORT: t->has_abort = 1; if (e->value == ABORT_ROUND) t->has_abort_round = 1; break;
                default: break;
            }
        }
        t->op_n = nops - t->op_lo;
        int writes = 0;
        for (uint64_t k = 0; k < t->op_n; ++k) writes += ops[t->op_lo + k]->kind == EV_WRITE;
        t->read_only = writes == 0;
        if (!t->device) t->key = 2 * t->key + t->read_only; /* RO right after the update that made its snapshot */
        /* incomplete: a speculative commit with no verdict, or an attempt still open */
        const int open = t->has_begin && !t->has_spec && !t->has_abort;
        if ((t->has_spec && !t->has_final && !t->has_abort_round) || open) {
            res->verdict = ORC_CHECK_INCOMPLETE;
            res->reason = ORC_REASON_INCOMPLETE;
            res->tx = t->id;
            goto out;
        }
    }
    /* ---- real time: host commit ts vs begin/commit order; device tickets vs batch order */
    {
        uint64_t nh = 0;
        for (uint64_t i = 0; i < nt; ++i)
            if (txs[i].has_final && !txs[i].device) order[nh++] = &txs[i];
        /* sweep by seq: (begin_seq, 0) and (spec_seq, 1) marks */
        mark* mk = malloc(2 * nh * sizeof *mk + 1);
        uint64_t nm = 0;
        for (uint64_t i = 0; i < nh; ++i) {
            mk[nm++] = (mark){order[i]->begin_seq, order[i], 0};
            mk[nm++] = (mark){order[i]->spec_seq, order[i], 1};
        }
        qsort(mk, nm, sizeof *mk, cmp_mark);
        uint64_t max_ts = 0; /* max commit ts of update txs committed so far */
        uint64_t* bound = calloc(nt, 8);
        for (uint64_t i = 0; i < nm; ++i) {
            txrec* t = mk[i].t;
            const uint64_t idx = (uint64_t)(t - txs);
            if (!mk[i].is_commit) bound[idx] = max_ts;
            else {
                const uint64_t ts = t->key >> 1;
                const int ok = t->read_only ? ts >= bound[idx] : ts > bound[idx];
                if (!ok && res->verdict == ORC_CHECK_PASS) {
                    res->verdict = ORC_CHECK_FAIL;
                    res->reason = ORC_REASON_REALTIME;
                    res->tx = t->id;
                    res->expected = bound[idx];
                    res->got = ts;
                    res->round = t->round;
                }
                if (!t->read_only && ts > max_ts) max_ts = ts;
            }
        }
        free(bound);
        free(mk);
        if (res->verdict != ORC_CHECK_PASS) goto out;
        /* device: within a round, ticket order must not invert batch order */
        uint64_t nd = 0;
        for (uint64_t i = 0; i < nt; ++i)
            if (txs[i].has_spec && txs[i].device) order[nd++] = &txs[i];
        qsort(order, nd, sizeof *order, cmp_claimed);
        for (uint64_t i = 1; i < nd; ++i)
            if (order[i]->round == order[i - 1]->round &&
                ((order[i]->id >> 32) & 0x7fffffffu) < ((order[i - 1]->id >> 32) & 0x7fffffffu)) {
                res->verdict = ORC_CHECK_FAIL;
                res->reason = ORC_REASON_REALTIME;
                res->tx = order[i]->id;
                res->round = order[i]->round;
                goto out;
            }
    }
    /* ---- replay rounds in claimed order */
    memcpy(state, init, words * 8);
    uint64_t nf = 0;
    for (uint64_t i = 0; i < nt; ++i)
        if (txs[i].has_spec && (txs[i].has_final || txs[i].has_abort_round)) order[nf++] = &txs[i];
    qsort(order, nf, sizeof *order, cmp_claimed);
    overlay ov = {0};
    if (want_p2 && !ov_init(&ov, 16 * nf)) {
        res->verdict = ORC_CHECK_INCOMPLETE;
        goto out;
    }
    for (uint64_t lo = 0; lo < nf;) {
        uint64_t hi = lo;
        while (hi < nf && order[hi]->round == order[lo]->round) ++hi;
        if (want_p2) { /* the aborted side(s) of this round, on the round-start state */
            for (int dev = 0; dev < 2; ++dev) {
                txrec **spec = malloc((hi - lo) * sizeof *spec), **extra = malloc((hi - lo) * sizeof *extra);
                uint64_t ns = 0, nx = 0;
                for (uint64_t i = lo; i < hi; ++i) {
                    if (order[i]->device == dev && !order[i]->has_final) spec[ns++] = order[i];
                    if (order[i]->device != dev && order[i]->has_final) extra[nx++] = order[i];
                }
                int bad = 0;
                if (ns) {
                    replay_ctx c = {ops, state, words, &ov, NULL, res, 1};
                    bad = check_spec_set(&c, spec, ns, extra, nx);
                }
                free(spec);
                free(extra);
                if (bad) goto out_ov;
            }
        } else { /* P1: the finally committed transactions in claimed order */
            replay_ctx c = {ops, state, words, NULL, state, res, 1};
            for (uint64_t i = lo; i < hi; ++i)
                if (order[i]->has_final && replay_tx(&c, order[i])) goto out_ov;
        }
        if (want_p2) { /* advance the committed state for the next round */
            orc_check_result scratch = *res;
            replay_ctx c = {ops, state, words, NULL, state, &scratch, 0};
            for (uint64_t i = lo; i < hi; ++i)
                if (order[i]->has_final) (void)replay_tx(&c, order[i]);
        }
        lo = hi;
    }
out_ov:
    if (want_p2) ov_free(&ov);
out:
    free(srt), free(ops), free(txs), free(order), free(state);
    return res->verdict;
}

int orc_check_p1(const orc_trace_event* ev, uint64_t n, const uint64_t* init, uint64_t words, orc_check_result* res) {
    return check_trace(ev, n, init, words, 0, res);
}

int orc_check_p2dagger(const orc_trace_event* ev, uint64_t n, const uint64_t* init, uint64_t words,
                       orc_check_result* res) {
    return check_trace(ev, n, init, words, 1, res);
}
