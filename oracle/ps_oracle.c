/*
 * ps_oracle.c — CPU restatement of the reference hot path.  TEST INFRASTRUCTURE ONLY (see header).
 *
 * Deliberately follows the reference's own algorithm and data layout choices rather than the
 * GPU design: a sorted (time, delta) ledger per stage with insort, an earliest_fit that rebuilds
 * merged usages and suffix maxima on every query and walks breakpoints, a derived-mode pending
 * refresh that scans every offloaded op each step, and makespan / peak recomputed from the event
 * lists afterwards.  Every function cites the reference lines it restates.
 */
#include "ps_oracle.h"

#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <pthread.h>
#include <unistd.h>

#define NONE_T INT64_MIN

typedef struct {
    int64_t t, d;
} point;

/* _MemLedger (listsched.py:52-60): committed (time, delta) points kept sorted. */
typedef struct {
    point *p;
    int n;
    int64_t limit;
} ledger;

/* insort(points, (time, delta)): insert after every tuple <= (t, d) (listsched.py:59-60). */
static void ledger_add(ledger *L, int64_t t, int64_t d) {
    int lo = 0, hi = L->n;
    while (lo < hi) {
        int mid = (lo + hi) / 2;
        if (L->p[mid].t < t || (L->p[mid].t == t && L->p[mid].d <= d)) lo = mid + 1;
        else hi = mid;
    }
    memmove(L->p + lo + 1, L->p + lo, (size_t)(L->n - lo) * sizeof(point));
    L->p[lo].t = t;
    L->p[lo].d = d;
    L->n++;
}

/* earliest_fit (listsched.py:62-100).  scratch holds 3*n int64. Returns NONE_T for None. */
static int64_t ledger_earliest_fit(const ledger *L, int64_t lo, int64_t delta, int64_t lag, int64_t *scratch) {
    if (delta <= 0) return lo;
    int64_t *times = scratch, *usages = scratch + L->n, *suffmax = scratch + 2 * L->n;
    int nb = 0;
    int64_t run = 0;
    for (int k = 0; k < L->n; ++k) {           /* usage after each breakpoint, merged (68-75) */
        run += L->p[k].d;
        if (nb && times[nb - 1] == L->p[k].t) {
            usages[nb - 1] = run;
        } else {
            times[nb] = L->p[k].t;
            usages[nb] = run;
            nb++;
        }
    }
    for (int k = 0; k < nb; ++k) suffmax[k] = usages[k];          /* suffix maxima (76-78) */
    for (int k = nb - 2; k >= 0; --k)
        if (suffmax[k + 1] > suffmax[k]) suffmax[k] = suffmax[k + 1];
    int64_t t = lo;
    for (;;) {
        /* worst_from(t + lag) (80-86) */
        int64_t T = t + lag;
        int a = 0, b = nb;
        while (a < b) {                        /* bisect_right(times, T) */
            int mid = (a + b) / 2;
            if (times[mid] <= T) a = mid + 1;
            else b = mid;
        }
        int64_t cur = a ? usages[a - 1] : 0;
        int64_t later = a < nb ? suffmax[a] : 0;
        int64_t worst = cur > later ? cur : later;
        if (worst + delta <= L->limit) return t;
        /* jump to the next breakpoint after t + lag (92-100) */
        int found = 0;
        for (int k = 0; k < nb; ++k)
            if (times[k] > T) {
                t = times[k] - lag;
                found = 1;
                break;
            }
        if (!found) return NONE_T;
    }
}

typedef struct {
    uint32_t code; /* (rank << 30) | (i << 24) | (j << 2) | kind */
    int64_t start, end;
} event;

typedef struct {
    const or_instance *I;
    int P, m, G, L;
    int64_t *done;        /* [P*m*3] end time or -1: st.done (listsched.py:106) */
    int64_t *off_end;     /* [P*m]  st.offload_end */
    int64_t *rel_end;     /* [P*m]  st.reload_end  */
    ledger *mem;          /* [P]    st.mem          */
    point *pool;
    int64_t *scratch;
} state;

#define OP(i, j, k) (((size_t)(i) * S->m + (j)) * 3 + (k))

/* _compute_ready (listsched.py:114-145). Returns NONE_T when a prerequisite is uncommitted. */
static int64_t compute_ready(const state *S, int i, int j, int k, const uint8_t *offl) {
    int64_t fl = 0;
    if (k == 0) {
        if (i > 0) {
            int64_t up = S->done[OP(i - 1, j, 0)];
            if (up < 0) return NONE_T;
            if (up + S->I->comm > fl) fl = up + S->I->comm;
        }
    } else if (k == 1) {
        int64_t own = S->done[OP(i, j, 0)];
        if (own < 0) return NONE_T;
        if (own > fl) fl = own;
        if (i < S->P - 1) {
            int64_t dn = S->done[OP(i + 1, j, 1)];
            if (dn < 0) return NONE_T;
            if (dn + S->I->comm > fl) fl = dn + S->I->comm;
        }
        if (offl[(size_t)i * S->m + j]) {
            int64_t r = S->rel_end[(size_t)i * S->m + j];
            if (r < 0) return NONE_T;
            if (r > fl) fl = r;
        }
    } else {
        int64_t own = S->done[OP(i, j, 1)];
        if (own < 0) return NONE_T;
        if (own > fl) fl = own;
    }
    return fl;
}

/* candidate key (time, rank, OpId) compared lexicographically (listsched.py:230-231, 243-245) */
typedef struct {
    int64_t t;
    int rank, i, j, k;
    int kind;   /* transfers: 0 offload, 1 reload; chan g */
    int g;
} cand;

static int cand_less(const cand *a, const cand *b) {
    if (a->t != b->t) return a->t < b->t;
    if (a->rank != b->rank) return a->rank < b->rank;
    if (a->i != b->i) return a->i < b->i;
    if (a->j != b->j) return a->j < b->j;
    return a->k < b->k;
}

int or_run_order(const or_instance *I, const uint16_t *orders, int32_t stride, const uint32_t *mask,
                 const uint32_t *chorders, int32_t cstride, or_result *out) {
    const int P = I->P, m = I->m, G = I->G, Lo = 3 * m;
    out->makespan = -1;
    out->bubble = 0.0;
    out->flags = 0;
    out->blocked = 0;
    out->n_events = 0;
    /* structural checks: every op code names an op of its stage (a row may be shorter than 3m —
     * terminated by OR_END — or repeat ops: run_order replays such rows literally, committing a
     * repeated op again, and ends in OrderInfeasible since some op is never committed,
     * listsched.py:206-252); offload bits only on offloadable F ops (KeyError in the reference) */
    uint8_t *offl = (uint8_t *)calloc((size_t)P * m, 1);
    int *row_len = (int *)malloc((size_t)P * sizeof(int));
    int n_off = 0, bad = 0;
    for (int i = 0; i < P && !bad; ++i) {
        row_len[i] = Lo;
        for (int q = 0; q < Lo; ++q) {
            uint32_t c = orders[(size_t)i * stride + q];
            if (c == OR_END) { row_len[i] = q; break; }
            uint32_t j = c >> 2, k = c & 3;
            if (j >= (uint32_t)m || k > 2) { bad = 1; break; }
        }
    }
    for (int b = 0; b < P * m; ++b)
        if ((mask[b >> 5] >> (b & 31)) & 1u) {
            if (I->act[b] <= 0) bad = 1;
            offl[b] = 1;
            n_off++;
        }
    if (bad) {
        free(row_len);
        free(offl);
        out->flags = 4;
        return 0;
    }

    state Sv;
    state *S = &Sv;
    S->I = I; S->P = P; S->m = m; S->G = G; S->L = Lo;
    size_t nops = (size_t)P * m * 3;
    S->done = (int64_t *)malloc(nops * sizeof(int64_t));
    S->off_end = (int64_t *)malloc((size_t)P * m * sizeof(int64_t));
    S->rel_end = (int64_t *)malloc((size_t)P * m * sizeof(int64_t));
    for (size_t k = 0; k < nops; ++k) S->done[k] = -1;
    for (size_t k = 0; k < (size_t)P * m; ++k) S->off_end[k] = S->rel_end[k] = -1;
    int cap = 5 * m + 8;
    S->mem = (ledger *)calloc((size_t)P, sizeof(ledger));
    S->pool = (point *)malloc((size_t)P * cap * sizeof(point));
    S->scratch = (int64_t *)malloc((size_t)3 * cap * sizeof(int64_t));
    for (int i = 0; i < P; ++i) {
        S->mem[i].p = S->pool + (size_t)i * cap;
        S->mem[i].limit = I->limit[i];
    }
    int *stage_pos = (int *)calloc((size_t)P, sizeof(int));
    int64_t *stage_free = (int64_t *)calloc((size_t)P, sizeof(int64_t));
    int64_t *chan_free = (int64_t *)calloc((size_t)G, sizeof(int64_t));
    int *chan_pos = (int *)calloc((size_t)G, sizeof(int));
    const int derived = chorders == NULL;
    /* derived mode: pending requests per channel, (x, kind) unsorted (listsched.py:180-181) */
    int *pend = (int *)malloc((size_t)G * 2 * P * m * sizeof(int));
    int *npend = (int *)calloc((size_t)G, sizeof(int));
    uint8_t *requested = (uint8_t *)calloc((size_t)P * m * 2, 1);
    event *evs = (event *)malloc((size_t)(nops + 2 * n_off + 1) * sizeof(event));
    int n_ev = 0;
    size_t total = nops, n_done = 0;
    int total_tr = 2 * n_off, n_tr = 0;

    while (n_done < total || n_tr < total_tr) {
        if (derived) {                                           /* refresh (207-214) */
            for (int x = 0; x < P * m; ++x) {
                if (!offl[x]) continue;
                int i = x / m;
                int g = I->chan[i];
                if (S->done[(size_t)x * 3] >= 0 && !requested[2 * x]) {
                    requested[2 * x] = 1;
                    pend[(size_t)g * 2 * P * m + npend[g]++] = 2 * x;       /* OFFLOAD */
                }
                if (S->off_end[x] >= 0 && !requested[2 * x + 1]) {
                    requested[2 * x + 1] = 1;
                    pend[(size_t)g * 2 * P * m + npend[g]++] = 2 * x + 1;   /* RELOAD */
                }
            }
        }
        cand best = {0, 0, 0, 0, 0, 0, 0};
        int have = 0;
        for (int i = 0; i < P; ++i) {                            /* stage heads (217-232) */
            if (stage_pos[i] >= row_len[i]) continue;
            uint32_t c = orders[(size_t)i * stride + stage_pos[i]];
            int j = (int)(c >> 2), k = (int)(c & 3);
            int64_t ready = compute_ready(S, i, j, k, offl);
            if (ready == NONE_T) continue;
            int64_t lo = ready > stage_free[i] ? ready : stage_free[i];
            if (k == 0) {
                lo = ledger_earliest_fit(&S->mem[i], lo, I->delta[OP(i, j, 0)], I->proc[OP(i, j, 0)], S->scratch);
                if (lo == NONE_T) continue;
            }
            cand cd = {lo, 0, i, j, k, 0, 0};
            if (!have || cand_less(&cd, &best)) { best = cd; have = 1; }
        }
        for (int g = 0; g < G; ++g) {                            /* channels (233-246) */
            int nopt;
            int opts_buf[1];
            const int *opts;
            if (derived) {
                opts = pend + (size_t)g * 2 * P * m;
                nopt = npend[g];
            } else {
                uint32_t e = chan_pos[g] < cstride ? chorders[(size_t)g * cstride + chan_pos[g]] : 0xFFFFFFFFu;
                nopt = 0;
                if (e != 0xFFFFFFFFu) {
                    int x = (int)((e >> 16) & 0x7FFF) * m + (int)(e & 0xFFFF);
                    opts_buf[0] = 2 * x + (int)(e >> 31);
                    nopt = 1;
                }
                opts = opts_buf;
            }
            for (int q = 0; q < nopt; ++q) {
                int x = opts[q] >> 1, reload = opts[q] & 1;
                int i = x / m, j = x % m;
                /* transfer_floor / transfer_candidate (186-204) */
                int64_t floor_t = reload ? S->off_end[x] : S->done[(size_t)x * 3];
                if (floor_t < 0) continue;
                int64_t lo = floor_t > chan_free[g] ? floor_t : chan_free[g];
                if (reload) {
                    lo = ledger_earliest_fit(&S->mem[i], lo, I->act[x], 0, S->scratch);
                    if (lo == NONE_T) continue;
                }
                cand cd = {lo, reload ? 1 : 2, i, j, 0, reload, g};
                if (!have || cand_less(&cd, &best)) { best = cd; have = 1; }
            }
        }
        if (!have) {                                             /* OrderInfeasible (248-252) */
            for (int i = 0; i < P; ++i)
                if (stage_pos[i] < row_len[i]) out->blocked |= 1u << i;
            out->flags = 2;
            break;
        }
        uint32_t code = ((uint32_t)best.rank << 30) | ((uint32_t)best.i << 24) | ((uint32_t)best.j << 2) | (uint32_t)best.k;
        if (best.rank == 0) {                                    /* _commit_compute (148-152, 255-259) */
            int64_t end = best.t + I->proc[OP(best.i, best.j, best.k)];
            if (S->done[OP(best.i, best.j, best.k)] >= 0) n_done--;     /* a repeated op: len(done) stays */
            S->done[OP(best.i, best.j, best.k)] = end;
            ledger_add(&S->mem[best.i], end, I->delta[OP(best.i, best.j, best.k)]);
            stage_pos[best.i]++;
            stage_free[best.i] = end;
            n_done++;
            evs[n_ev].code = code; evs[n_ev].start = best.t; evs[n_ev].end = end; n_ev++;
        } else {                                                 /* _commit_transfer (155-164, 260-267) */
            int x = best.i * m + best.j;
            int64_t end = best.t + I->toff;
            int64_t gamma = I->act[x];
            if (!best.kind) {
                S->off_end[x] = end;
                ledger_add(&S->mem[best.i], end, -gamma);
            } else {
                S->rel_end[x] = end;
                ledger_add(&S->mem[best.i], best.t, gamma);
            }
            chan_free[best.g] = end;
            if (derived) {
                int *pl = pend + (size_t)best.g * 2 * P * m;
                for (int q = 0; q < npend[best.g]; ++q)
                    if (pl[q] == 2 * x + best.kind) {
                        pl[q] = pl[--npend[best.g]];
                        break;
                    }
            } else {
                chan_pos[best.g]++;
            }
            n_tr++;
            evs[n_ev].code = code; evs[n_ev].start = best.t; evs[n_ev].end = end; n_ev++;
        }
    }

    if (out->flags != 2) {
        out->flags = 1;
        /* makespan (schedule.py:168-183) from the compute events */
        int64_t span;
        if (I->post) {
            span = 0;
            for (int i = 0; i < P; ++i) {
                int64_t f0 = INT64_MAX, w1 = INT64_MIN;
                for (int e = 0; e < n_ev; ++e) {
                    uint32_t c = evs[e].code;
                    if ((c >> 30) || (int)((c >> 24) & 63) != i) continue;
                    if ((c & 3) == 0 && evs[e].start < f0) f0 = evs[e].start;
                    if ((c & 3) == 2 && evs[e].end > w1) w1 = evs[e].end;
                }
                if (w1 - f0 > span) span = w1 - f0;
            }
        } else {
            int64_t hi = INT64_MIN, lo = INT64_MAX;
            for (int e = 0; e < n_ev; ++e) {
                if (evs[e].code >> 30) continue;
                if (evs[e].end > hi) hi = evs[e].end;
                if (evs[e].start < lo) lo = evs[e].start;
            }
            span = hi - lo;
        }
        out->makespan = span;
        int64_t busy = 0;
        for (size_t k = 0; k < nops; ++k) busy += I->proc[k];
        out->bubble = 1.0 - (double)busy / ((double)P * (double)span);   /* cli.py:156 unrounded */
        if (out->peak) {
            /* memory_trace STRICT (schedule.py:188-237): per stage, merge equal times, prefix-sum */
            point *pts = (point *)malloc((size_t)(n_ev + 1) * sizeof(point));
            for (int i = 0; i < P; ++i) {
                int np = 0;
                for (int e = 0; e < n_ev; ++e) {
                    uint32_t c = evs[e].code;
                    if ((int)((c >> 24) & 63) != i) continue;
                    int rank = (int)(c >> 30), j = (int)((c >> 2) & 0x3FFFFF), k = (int)(c & 3);
                    if (rank == 0) { pts[np].t = evs[e].end; pts[np].d = I->delta[OP(i, j, k)]; }
                    else if (rank == 1) { pts[np].t = evs[e].start; pts[np].d = I->act[(size_t)i * m + j]; }
                    else { pts[np].t = evs[e].end; pts[np].d = -I->act[(size_t)i * m + j]; }
                    np++;
                }
                /* insertion sort by time (stable), then merged replay */
                for (int a = 1; a < np; ++a) {
                    point v = pts[a];
                    int b = a - 1;
                    while (b >= 0 && pts[b].t > v.t) { pts[b + 1] = pts[b]; --b; }
                    pts[b + 1] = v;
                }
                int64_t usage = 0, peak = 0;
                for (int a = 0; a < np;) {
                    int64_t t = pts[a].t, sum = 0;
                    while (a < np && pts[a].t == t) sum += pts[a++].d;
                    if (sum == 0) continue;
                    usage += sum;
                    if (usage > peak) peak = usage;
                }
                out->peak[i] = peak;
            }
            free(pts);
        }
    }
    if (out->trace_code)
        for (int e = 0; e < n_ev; ++e) {
            out->trace_code[e] = evs[e].code;
            out->trace_start[e] = (int32_t)evs[e].start;
        }
    out->n_events = n_ev;

    free(offl); free(row_len); free(S->done); free(S->off_end); free(S->rel_end); free(S->mem); free(S->pool);
    free(S->scratch); free(stage_pos); free(stage_free); free(chan_free); free(chan_pos); free(pend);
    free(npend); free(requested); free(evs);
    return 0;
}

/* Work splitting over host threads (pthreads; the image has no OpenMP runtime). */
typedef struct {
    int64_t next, n;
    pthread_mutex_t mu;
    void (*body)(void *ctx, int64_t c, void *tls);
    void *(*tls_new)(void *ctx);
    void (*tls_done)(void *ctx, void *tls);
    void *ctx;
} pool;

static void *pool_worker(void *arg) {
    pool *pl = (pool *)arg;
    void *tls = pl->tls_new ? pl->tls_new(pl->ctx) : NULL;
    for (;;) {
        pthread_mutex_lock(&pl->mu);
        int64_t c = pl->next++;
        pthread_mutex_unlock(&pl->mu);
        if (c >= pl->n) break;
        pl->body(pl->ctx, c, tls);
    }
    if (pl->tls_done) pl->tls_done(pl->ctx, tls);
    return NULL;
}

static void pool_run(int threads, int64_t n, void (*body)(void *, int64_t, void *), void *(*tls_new)(void *),
                     void (*tls_done)(void *, void *), void *ctx) {
    if (threads <= 0) threads = (int)sysconf(_SC_NPROCESSORS_ONLN);
    if (threads < 1) threads = 1;
    if (threads > n) threads = (int)(n > 0 ? n : 1);
    pool pl;
    pl.next = 0; pl.n = n; pl.body = body; pl.tls_new = tls_new; pl.tls_done = tls_done; pl.ctx = ctx;
    pthread_mutex_init(&pl.mu, NULL);
    pthread_t *th = (pthread_t *)malloc((size_t)threads * sizeof(pthread_t));
    for (int t = 1; t < threads; ++t) pthread_create(&th[t], NULL, pool_worker, &pl);
    pool_worker(&pl);
    for (int t = 1; t < threads; ++t) pthread_join(th[t], NULL);
    free(th);
    pthread_mutex_destroy(&pl.mu);
}

typedef struct {
    const or_instance *I;
    const uint16_t *orders;
    int32_t stride;
    const uint32_t *masks;
    int32_t mask_words;
    const uint32_t *chorders;
    int32_t cstride;
    int64_t *makespan, *peak;
    double *bubble;
    uint32_t *flags, *blocked;
} batch_ctx;

static void batch_body(void *vctx, int64_t c, void *tls) {
    batch_ctx *b = (batch_ctx *)vctx;
    (void)tls;
    or_result r;
    memset(&r, 0, sizeof r);
    r.peak = b->peak ? b->peak + c * b->I->P : NULL;
    or_run_order(b->I, b->orders + (size_t)c * b->I->P * b->stride, b->stride, b->masks + (size_t)c * b->mask_words,
                 b->chorders ? b->chorders + (size_t)c * b->I->G * b->cstride : NULL, b->cstride, &r);
    b->makespan[c] = r.makespan;
    if (b->bubble) b->bubble[c] = r.bubble;
    b->flags[c] = r.flags;
    if (b->blocked) b->blocked[c] = r.blocked;
}

int or_eval_batch(const or_instance *I, int64_t N, const uint16_t *orders, int32_t stride,
                  const uint32_t *masks, int32_t mask_words, const uint32_t *chorders, int32_t cstride,
                  int64_t *makespan, double *bubble, int64_t *peak, uint32_t *flags, uint32_t *blocked,
                  int32_t threads) {
    batch_ctx b = {I, orders, stride, masks, mask_words, chorders, cstride, makespan, peak, bubble, flags, blocked};
    pool_run(threads, N, batch_body, NULL, NULL, &b);
    return 0;
}

/* Philox4x32-10 (Salmon et al., SC'11; Random123 constants). */
void or_philox4x32_10(const uint32_t ctr[4], const uint32_t key[2], uint32_t out[4]) {
    uint32_t c0 = ctr[0], c1 = ctr[1], c2 = ctr[2], c3 = ctr[3], k0 = key[0], k1 = key[1];
    for (int r = 0; r < 10; ++r) {
        if (r) { k0 += 0x9E3779B9u; k1 += 0xBB67AE85u; }
        uint64_t p0 = (uint64_t)0xD2511F53u * c0, p1 = (uint64_t)0xCD9E8D57u * c2;
        uint32_t n0 = (uint32_t)(p1 >> 32) ^ c1 ^ k0, n2 = (uint32_t)(p0 >> 32) ^ c3 ^ k1;
        c0 = n0; c1 = (uint32_t)p1; c2 = n2; c3 = (uint32_t)p0;
    }
    out[0] = c0; out[1] = c1; out[2] = c2; out[3] = c3;
}

/* neighbour = incumbent + one move decoded from Philox(index, round; seed). */
int or_neighbour(const or_instance *I, const uint16_t *inc, int32_t stride, const uint32_t *inc_mask,
                 const or_moves *mv, uint64_t round, uint64_t index, uint16_t *out, uint32_t *mask_out) {
    const int P = I->P, m = I->m, Lo = 3 * m;
    int mask_words = (P * m + 31) / 32;
    memcpy(out, inc, (size_t)P * stride * sizeof(uint16_t));
    memcpy(mask_out, inc_mask, (size_t)mask_words * sizeof(uint32_t));
    uint32_t ctr[4] = {(uint32_t)index, (uint32_t)(index >> 32), (uint32_t)round, (uint32_t)(round >> 32)};
    uint32_t key[2] = {(uint32_t)mv->seed, (uint32_t)(mv->seed >> 32)};
    uint32_t r[4];
    or_philox4x32_10(ctr, key, r);
    int any_off = 0;
    for (int k = 0; k < P * m; ++k)
        if (I->act[k] > 0) { any_off = 1; break; }
    int s = (int)(r[1] % (uint32_t)P);
    if (!any_off || r[0] % 1000u < mv->shift_permille) {
        int a = (int)(r[2] % (uint32_t)Lo);
        uint32_t D = mv->max_shift ? mv->max_shift : 1u;
        int d = 1 + (int)((r[3] >> 1) % D);
        int b = (r[3] & 1u) ? a - d : a + d;
        if (b < 0) b = 0;
        if (b > Lo - 1) b = Lo - 1;
        if (b == a) return 0;
        uint16_t *row = out + (size_t)s * stride;
        uint16_t v = row[a];
        if (a < b) memmove(row + a, row + a + 1, (size_t)(b - a) * sizeof(uint16_t));
        else memmove(row + b + 1, row + b, (size_t)(a - b) * sizeof(uint16_t));
        row[b] = v;
        return 1;
    }
    int j = (int)(r[2] % (uint32_t)m);
    if (I->act[(size_t)s * m + j] <= 0) return 0;
    int bit = s * m + j;
    mask_out[bit >> 5] ^= 1u << (bit & 31);
    return 2;
}

/* Channel-order neighbour: the search over explicit channel orders.  A stage-op
 * SHIFT exactly as or_neighbour when r0 % 1000 < shift_permille (or no channel carries a
 * transfer); otherwise RSHIFT: channel g = r1 % G, the transfer at position a = r2 % len_g moves
 * to b = a -/+ d (d = 1 + (r3 >> 1) % max_shift, clamped), len_g = entries before the first
 * 0xFFFFFFFF pad.  Offload bits never change.  Returns 0 no-op, 1 SHIFT, 3 RSHIFT. */
int or_neighbour_explicit(const or_instance *I, const uint16_t *inc, int32_t stride, const uint32_t *inc_mask,
                          const uint32_t *inc_chan, int32_t cstride, const or_moves *mv, uint64_t round,
                          uint64_t index, uint16_t *out, uint32_t *mask_out, uint32_t *chan_out) {
    const int P = I->P, m = I->m, G = I->G, Lo = 3 * m;
    memcpy(out, inc, (size_t)P * stride * sizeof(uint16_t));
    memcpy(mask_out, inc_mask, (size_t)((P * m + 31) / 32) * sizeof(uint32_t));
    memcpy(chan_out, inc_chan, (size_t)G * cstride * sizeof(uint32_t));
    int total = 0;
    for (int g = 0; g < G; ++g)
        for (int q = 0; q < cstride && inc_chan[(size_t)g * cstride + q] != 0xFFFFFFFFu; ++q) total++;
    uint32_t ctr[4] = {(uint32_t)index, (uint32_t)(index >> 32), (uint32_t)round, (uint32_t)(round >> 32)};
    uint32_t key[2] = {(uint32_t)mv->seed, (uint32_t)(mv->seed >> 32)};
    uint32_t r[4];
    or_philox4x32_10(ctr, key, r);
    const uint32_t D = mv->max_shift ? mv->max_shift : 1u;
    if (total == 0 || r[0] % 1000u < mv->shift_permille) {
        int s = (int)(r[1] % (uint32_t)P);
        int a = (int)(r[2] % (uint32_t)Lo);
        int d = 1 + (int)((r[3] >> 1) % D);
        int b = (r[3] & 1u) ? a - d : a + d;
        if (b < 0) b = 0;
        if (b > Lo - 1) b = Lo - 1;
        if (b == a) return 0;
        uint16_t *row = out + (size_t)s * stride;
        uint16_t v = row[a];
        if (a < b) memmove(row + a, row + a + 1, (size_t)(b - a) * sizeof(uint16_t));
        else memmove(row + b + 1, row + b, (size_t)(a - b) * sizeof(uint16_t));
        row[b] = v;
        return 1;
    }
    int g = (int)(r[1] % (uint32_t)G);
    int len = 0;
    while (len < cstride && inc_chan[(size_t)g * cstride + len] != 0xFFFFFFFFu) len++;
    if (len < 2) return 0;
    int a = (int)(r[2] % (uint32_t)len);
    int d = 1 + (int)((r[3] >> 1) % D);
    int b = (r[3] & 1u) ? a - d : a + d;
    if (b < 0) b = 0;
    if (b > len - 1) b = len - 1;
    if (b == a) return 0;
    uint32_t *row = chan_out + (size_t)g * cstride;
    uint32_t v = row[a];
    if (a < b) memmove(row + a, row + a + 1, (size_t)(b - a) * sizeof(uint32_t));
    else memmove(row + b + 1, row + b, (size_t)(a - b) * sizeof(uint32_t));
    row[b] = v;
    return 3;
}

typedef struct {
    const or_instance *I;
    const uint16_t *inc;
    int32_t stride;
    const uint32_t *inc_mask;
    const uint32_t *inc_chan;   /* explicit channel-order search when non-NULL */
    int32_t cstride;
    const or_moves *mv;
    uint64_t round;
    int64_t first;
    int64_t *makespans;
    int64_t best;
    pthread_mutex_t mu;
} search_ctx;

typedef struct {
    uint16_t *ord;
    uint32_t *msk;
    uint32_t *chn;
    int64_t best;
} search_tls;

static void *search_tls_new(void *vctx) {
    search_ctx *s = (search_ctx *)vctx;
    search_tls *t = (search_tls *)malloc(sizeof(search_tls));
    t->ord = (uint16_t *)malloc((size_t)s->I->P * s->stride * sizeof(uint16_t));
    t->msk = (uint32_t *)malloc((size_t)((s->I->P * s->I->m + 31) / 32) * sizeof(uint32_t));
    t->chn = s->inc_chan ? (uint32_t *)malloc((size_t)s->I->G * s->cstride * sizeof(uint32_t)) : NULL;
    t->best = INT64_MAX;
    return t;
}

static void search_tls_done(void *vctx, void *vt) {
    search_ctx *s = (search_ctx *)vctx;
    search_tls *t = (search_tls *)vt;
    pthread_mutex_lock(&s->mu);
    if (t->best < s->best) s->best = t->best;
    pthread_mutex_unlock(&s->mu);
    free(t->ord);
    free(t->msk);
    free(t->chn);
    free(t);
}

static void search_body(void *vctx, int64_t c, void *vt) {
    search_ctx *s = (search_ctx *)vctx;
    search_tls *t = (search_tls *)vt;
    if (s->inc_chan)
        or_neighbour_explicit(s->I, s->inc, s->stride, s->inc_mask, s->inc_chan, s->cstride, s->mv, s->round,
                              (uint64_t)(s->first + c), t->ord, t->msk, t->chn);
    else
        or_neighbour(s->I, s->inc, s->stride, s->inc_mask, s->mv, s->round, (uint64_t)(s->first + c), t->ord, t->msk);
    or_result r;
    memset(&r, 0, sizeof r);
    or_run_order(s->I, t->ord, s->stride, t->msk, t->chn, s->inc_chan ? s->cstride : 0, &r);
    if (s->makespans) s->makespans[c] = r.flags == 1 ? r.makespan : -1;
    if (r.flags == 1) {
        int64_t key = (r.makespan << 32) | (int64_t)(uint32_t)(s->first + c);
        if (key < t->best) t->best = key;
    }
}

int64_t or_search_round(const or_instance *I, const uint16_t *inc, int32_t stride, const uint32_t *inc_mask,
                        const or_moves *mv, uint64_t round, int64_t first, int64_t count, int64_t *makespans,
                        int32_t threads) {
    return or_search_round_explicit(I, inc, stride, inc_mask, NULL, 0, mv, round, first, count, makespans, threads);
}

int64_t or_search_round_explicit(const or_instance *I, const uint16_t *inc, int32_t stride, const uint32_t *inc_mask,
                                 const uint32_t *inc_chan, int32_t cstride, const or_moves *mv, uint64_t round,
                                 int64_t first, int64_t count, int64_t *makespans, int32_t threads) {
    search_ctx s;
    s.I = I; s.inc = inc; s.stride = stride; s.inc_mask = inc_mask; s.mv = mv; s.round = round;
    s.inc_chan = inc_chan; s.cstride = cstride;
    s.first = first; s.makespans = makespans; s.best = INT64_MAX;
    pthread_mutex_init(&s.mu, NULL);
    pool_run(threads, count, search_body, search_tls_new, search_tls_done, &s);
    pthread_mutex_destroy(&s.mu);
    return s.best;
}

/* ---- B&B node lower bound: solver._Search._bound (solver.py:352-383) with _chain_ends
 * (solver.py:321-350), restated over dense tables.  start[(i*m + j)*3 + k] is the committed start
 * of op (i, j, k) or -1; sfree[i] the stage free time; t the node's clock. */
int64_t or_bound(const or_instance *I, int64_t t, const int64_t *sfree, const int64_t *start, int32_t post) {
    const int P = I->P, m = I->m;
#define ST(i, j, k) start[((size_t)(i) * m + (j)) * 3 + (k)]
#define PT(i, j, k) I->proc[((size_t)(i) * m + (j)) * 3 + (k)]
    if (post) {                                                    /* solver.py:354-369 */
        int64_t worst = 0;
        for (int i = 0; i < P; ++i) {
            int64_t rem = 0, first_f = INT64_MAX, last_w = INT64_MIN;
            int have_f = 0;
            for (int j = 0; j < m; ++j)
                for (int k = 0; k < 3; ++k) {
                    if (ST(i, j, k) < 0) { rem += PT(i, j, k); continue; }
                    if (k == 0) { have_f = 1; if (ST(i, j, 0) < first_f) first_f = ST(i, j, 0); }
                    if (k == 2 && ST(i, j, 2) + PT(i, j, 2) > last_w) last_w = ST(i, j, 2) + PT(i, j, 2);
                }
            int64_t v;
            if (rem == 0) v = last_w - first_f;
            else if (have_f) v = (sfree[i] > t ? sfree[i] : t) + rem - first_f;
            else v = rem;
            if (v > worst) worst = v;
        }
        return worst;
    }
    int64_t lb = 0, min_start = INT64_MAX;                         /* solver.py:370-383 */
    int any = 0;
    for (int i = 0; i < P; ++i)
        for (int j = 0; j < m; ++j)
            for (int k = 0; k < 3; ++k)
                if (ST(i, j, k) >= 0) {
                    any = 1;
                    if (ST(i, j, k) + PT(i, j, k) > lb) lb = ST(i, j, k) + PT(i, j, k);
                    if (ST(i, j, k) < min_start) min_start = ST(i, j, k);
                }
    for (int i = 0; i < P; ++i) {
        int64_t rem = 0;
        for (int j = 0; j < m; ++j)
            for (int k = 0; k < 3; ++k)
                if (ST(i, j, k) < 0) rem += PT(i, j, k);
        if (rem) {
            int64_t v = (sfree[i] > t ? sfree[i] : t) + rem;
            if (v > lb) lb = v;
        }
    }
    /* _chain_ends: F down the stages, then B up the stages with each W after its B */
    int64_t *E = (int64_t *)malloc(sizeof(int64_t) * (size_t)P * m * 3);
#define EE(i, j, k) E[((size_t)(i) * m + (j)) * 3 + (k)]
    for (int j = 0; j < m; ++j)
        for (int i = 0; i < P; ++i) {
            if (ST(i, j, 0) >= 0) { EE(i, j, 0) = ST(i, j, 0) + PT(i, j, 0); continue; }
            int64_t lo = sfree[i] > t ? sfree[i] : t;
            if (i > 0 && EE(i - 1, j, 0) + I->comm > lo) lo = EE(i - 1, j, 0) + I->comm;
            EE(i, j, 0) = lo + PT(i, j, 0);
        }
    for (int j = 0; j < m; ++j)
        for (int i = P - 1; i >= 0; --i) {
            if (ST(i, j, 1) >= 0) EE(i, j, 1) = ST(i, j, 1) + PT(i, j, 1);
            else {
                int64_t lo = sfree[i] > t ? sfree[i] : t;
                if (EE(i, j, 0) > lo) lo = EE(i, j, 0);
                if (i < P - 1 && EE(i + 1, j, 1) + I->comm > lo) lo = EE(i + 1, j, 1) + I->comm;
                EE(i, j, 1) = lo + PT(i, j, 1);
            }
            if (ST(i, j, 2) >= 0) EE(i, j, 2) = ST(i, j, 2) + PT(i, j, 2);
            else {
                int64_t lo = sfree[i] > t ? sfree[i] : t;
                if (EE(i, j, 1) > lo) lo = EE(i, j, 1);
                EE(i, j, 2) = lo + PT(i, j, 2);
            }
        }
    for (size_t q = 0; q < (size_t)P * m * 3; ++q)
        if (E[q] > lb) lb = E[q];
    free(E);
    if (any) lb -= min_start;
    return lb;
#undef EE
#undef ST
#undef PT
}
