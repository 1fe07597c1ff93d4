/*
 * ps_oracle.h — CPU restatement of the reference hot path.  TEST INFRASTRUCTURE ONLY.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference leg may load
 * this library, and only as the checker (or the timed CPU baseline) — never as the product path.
 *
 * Restates, function by function, /root/reference/pkg/src/pipesched:
 *   or_run_order      listsched.run_order        listsched.py:167-269 (incl. _MemLedger 52-100,
 *                                                _compute_ready 114-145, commits 148-164)
 *   and afterwards, from its event lists (still inside or_run_order):
 *     makespan        schedule.makespan          schedule.py:168-183
 *     peaks           schedule.memory_trace      schedule.py:188-237 (STRICT)
 *     bubble          cli._compare_row           cli.py:115, 156 (unrounded)
 * and, for the local search that has no reference counterpart, the normative move definition of
 * DESIGN.md §4 (Philox4x32-10 keyed by seed/round/index).
 *
 * Parity pinned against the reference: the JSON fixtures under tests/golden were produced by the
 * reference itself (tests/golden/make_golden.py); tests/test_oracle.py checks this restatement
 * against them.
 * Encodings are those of include/pipesched_b200.h.
 */
#ifndef PS_ORACLE_H
#define PS_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* stage-row terminator: a row shorter than 3m ends at the first OR_END (include/pipesched_b200.h
 * PS_ROW_END) */
#define OR_END 0xFFFFu

typedef struct or_instance {
    int32_t P, m, G;
    const int64_t *proc;      /* [P][m][3] */
    const int64_t *delta;     /* [P][m][3] */
    const int64_t *act;       /* [P][m]    */
    const int64_t *limit;     /* [P]       */
    const int32_t *chan;      /* [P]       */
    int64_t comm, toff;
    int32_t post;
} or_instance;

typedef struct or_result {
    int64_t makespan;         /* -1 unless feasible */
    double bubble;
    int64_t *peak;            /* [P] (optional) */
    uint32_t flags;           /* 1 feasible, 2 deadlock, 4 malformed */
    uint32_t blocked;         /* deadlock: stages with remaining ops */
    uint32_t *trace_code;     /* [>= 5Pm] (optional) */
    int32_t *trace_start;     /* [>= 5Pm] (optional) */
    int32_t n_events;
} or_result;

typedef struct or_moves {
    uint64_t seed;
    uint32_t shift_permille;
    uint32_t max_shift;
} or_moves;

/* One candidate. orders [P][stride] op codes, mask [ceil(P*m/32)], chorders [G][cstride] or NULL. */
int or_run_order(const or_instance *I, const uint16_t *orders, int32_t stride, const uint32_t *mask,
                 const uint32_t *chorders, int32_t cstride, or_result *out);

/* Batch over N candidates with `threads` OpenMP threads (0 = all); arrays of N results. */
int or_eval_batch(const or_instance *I, int64_t N, const uint16_t *orders, int32_t stride,
                  const uint32_t *masks, int32_t mask_words, const uint32_t *chorders, int32_t cstride,
                  int64_t *makespan, double *bubble, int64_t *peak, uint32_t *flags, uint32_t *blocked,
                  int32_t threads);

void or_philox4x32_10(const uint32_t ctr[4], const uint32_t key[2], uint32_t out[4]);

/* Neighbour `index` of round `round` applied to a copy of the incumbent (orders_out [P][stride],
   mask_out [mask_words]). Returns the move type (0 noop, 1 shift, 2 toggle). */
int or_neighbour(const or_instance *I, const uint16_t *inc_orders, int32_t stride, const uint32_t *inc_mask,
                 const or_moves *mv, uint64_t round, uint64_t index, uint16_t *orders_out, uint32_t *mask_out);

/* One local-search round on the CPU: evaluate neighbours [first, first+count), return the best
   key (makespan << 32 | index) or INT64_MAX; makespans (optional) receives each neighbour's. */
int64_t or_search_round(const or_instance *I, const uint16_t *inc_orders, int32_t stride,
                        const uint32_t *inc_mask, const or_moves *mv, uint64_t round, int64_t first,
                        int64_t count, int64_t *makespans, int32_t threads);

/* The channel-order search: neighbours of an incumbent with explicit channel
 * orders [G][cstride] (0xFFFFFFFF padded); stage-op shifts and transfer shifts within a channel. */
int or_neighbour_explicit(const or_instance *I, const uint16_t *inc_orders, int32_t stride, const uint32_t *inc_mask,
                          const uint32_t *inc_chan, int32_t cstride, const or_moves *mv, uint64_t round,
                          uint64_t index, uint16_t *orders_out, uint32_t *mask_out, uint32_t *chan_out);
int64_t or_search_round_explicit(const or_instance *I, const uint16_t *inc_orders, int32_t stride,
                                 const uint32_t *inc_mask, const uint32_t *inc_chan, int32_t cstride,
                                 const or_moves *mv, uint64_t round, int64_t first, int64_t count,
                                 int64_t *makespans, int32_t threads);

/* B&B node lower bound (solver.py:321-383): start [P][m][3] committed compute starts (-1 = not
   committed), sfree [P] stage free times, t the node clock, post the post-validation flag. */
int64_t or_bound(const or_instance *I, int64_t t, const int64_t *sfree, const int64_t *start, int32_t post);

#ifdef __cplusplus
}
#endif
#endif
