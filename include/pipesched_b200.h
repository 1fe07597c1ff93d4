/*
 * pipesched_b200.h — C ABI of the B200 candidate-schedule evaluator.
 *
 * Drop-in boundary for the reference hot path:
 *
 *   ps_eval_batch      replaces  listsched.run_order            (pkg/src/pipesched/listsched.py:167-269)
 *                      followed by schedule.makespan            (schedule.py:168-183),
 *                      schedule.memory_trace(STRICT).peak       (schedule.py:227-237)
 *                      and the bubble ratio                     (cli.py:115, 156),
 *                      for a whole batch of candidate structures at once.
 *   ps_eval_batch_host the same call on HOST buffers (copies in and out inside the call).
 *   ps_search_round_sharded  the same over G ranks: + one 8-byte NCCL all-reduce(MIN) per round
 *   ps_search_round    neighbour generation + evaluation + best-of selection of one local-search
 *                      round (no reference counterpart: SURVEY.md §0 "Not in the reference");
 *                      its result feeds solver.start_session(warm=...) (solver.py:543-565).
 *   ps_instance_create replaces the dict-keyed PipelineInstance tables (instance.py:62-177)
 *                      with dense, device-resident tables.
 *
 * Conventions (all indices 0-based here; the Python layer converts from the reference's 1-based
 * OpId(stage, microbatch, kind)):
 *   op code within a stage   (j << 2) | kind,  kind F=0, B=1, W=2        (instance.py:32-59)
 *   offload mask bit         i*m + j   (bit b lives in word b>>5, position b&31)
 *   channel-order entry      (kind << 31) | (i << 16) | j, kind 0=OFFLOAD 1=RELOAD; 0xFFFFFFFF pads
 *   trace entry              (rank << 30) | (i << 24) | (j << 2) | kind,
 *                            rank 0 = compute, 1 = reload, 2 = offload   (listsched.py:230, 243)
 *
 * Errors never cross the ABI as exceptions: functions return PS_OK or a negative PS_ERR_* code and
 * ps_last_error() describes the last failure on the calling thread.  Per-candidate outcomes
 * (deadlock = the reference's OrderInfeasible, listsched.py:248-252; malformed structure) are
 * reported in the flags array, never as call errors.
 *
 * Threading: an instance handle is immutable after creation and may be shared by threads and
 * streams; every call is asynchronous on the given stream except ps_instance_create/destroy and
 * ps_eval_batch_host.  Device pointers in the batch/result structs are owned by the caller.
 */
#ifndef PIPESCHED_B200_H
#define PIPESCHED_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PS_OK 0
#define PS_ERR_INVALID (-1)     /* bad argument or instance invariant broken            */
#define PS_ERR_RANGE (-2)       /* instance exceeds a supported size / value range     */
#define PS_ERR_CUDA (-3)        /* CUDA runtime error (see ps_last_error)              */
#define PS_ERR_NOMEM (-4)       /* device allocation failed                            */

#define PS_FLAG_FEASIBLE 1u     /* complete schedule; STRICT peak <= limit by construction */
#define PS_FLAG_DEADLOCK 2u     /* no event can start: the reference raises OrderInfeasible */
#define PS_FLAG_MALFORMED 4u    /* an op code names no op of its stage / bad offload bit / bad channel order */
#define PS_FLAG_RANGE 16u       /* an event time reached 2^29 quanta: search rounds drop the neighbour;
                                   ps_eval_batch finishes it in 64-bit time and keeps the flag only
                                   when a trace was requested and a time passes 2^31 - 1            */

/* Stage rows: 3m op codes (microbatch << 2 | kind), or fewer ending with PS_ROW_END (0xFFFF;
   0xFF for uint8 codes).  A row that repeats an op or is short is replayed literally, as the
   reference does (listsched.py:206-252): it ends in PS_FLAG_DEADLOCK with the blocked stages. */
#define PS_ROW_END 0xFFFFu

#define PS_MAX_STAGES 32
#define PS_MAX_MICROBATCHES 4096

typedef struct ps_instance ps_instance;
/* A recorded base candidate: its simulation checkpointed every few steps, so candidates that share
   a prefix of decisions with it resume from the last checkpoint before they diverge (exact; see
   DESIGN.md §3.5).  Created per instance, re-recorded whenever the base changes. */
typedef struct ps_base ps_base;

/* Dense instance tables, host memory, copied by ps_instance_create. */
typedef struct ps_instance_desc {
    int32_t num_stages;            /* P, 1..PS_MAX_STAGES                                      */
    int32_t num_microbatches;      /* m, 1..PS_MAX_MICROBATCHES                                */
    const int64_t *proc_time;      /* [P][m][3] compute durations (F,B,W), > 0                 */
    const int64_t *mem_delta;      /* [P][m][3] bytes; F > 0, B < 0, W < 0, sum 0             */
    const int64_t *act_size;       /* [P][m] offloadable bytes of the F activation, 0 = none */
    const int64_t *mem_limit;      /* [P] bytes, > 0                                           */
    const int32_t *stage_channel;  /* [P] transfer channel of each stage (topology group)      */
    int32_t num_channels;          /* G                                                        */
    int64_t comm_time;             /* >= 0                                                     */
    int64_t offload_time;          /* >= 0                                                     */
    int32_t post_validation;       /* 1: makespan = max over stages (last W end - first F start) */
} ps_instance_desc;

/* Layout facts callers need to size candidate / result buffers. */
typedef struct ps_instance_info {
    int32_t num_stages;
    int32_t num_microbatches;
    int32_t order_stride;          /* u16 entries per stage row of stage_orders (>= 3m, mult. of 8) */
    int32_t mask_words;            /* u32 words of one candidate's offload mask                    */
    int32_t max_events;            /* 5*P*m: trace_stride lower bound                              */
    int32_t value_bits;            /* 32 or 64: width of the device memory ledger                  */
    int64_t memory_unit;           /* gcd of all byte quantities (device ledger counts in these)   */
    int64_t busy_time;             /* sum of all proc_time (bubble numerator)                      */
    int32_t lanes_per_candidate;   /* warp lanes that evaluate one candidate (one per stage)        */
    int32_t device;
} ps_instance_info;

/* A batch of candidate structures, device memory. */
typedef struct ps_cand_batch {
    int64_t num_candidates;
    const void *stage_orders;       /* [N][P][order_stride] op codes, each row a permutation of the
                                       stage's 3m ops; uint16 codes, or uint8 (order_bytes = 1)    */
    const uint32_t *offload_mask;   /* [N][mask_words]                                               */
    const uint32_t *channel_orders; /* [N][G][chan_stride] or NULL = derived (greedy) channel mode   */
    int32_t chan_stride;
    const ps_base *base;            /* optional recorded base (derived mode, no trace): shared
                                       prefixes are restored instead of re-simulated            */
    int32_t order_bytes;            /* 2 (or 0): uint16 op codes; 1: uint8 op codes (m <= 64), half
                                       the bytes to move — what ps_eval_batch_host copies in    */
} ps_cand_batch;

/* Candidates as differences from one reference structure (host memory): the compact form of a
   batch of neighbours — a candidate that differs from `ref` in d stage-order positions and f
   offload bits costs 8d + 4f + 8 bytes instead of P*order_stride*2 + mask_words*4.
   Candidate c = ref with orders[stage][pos] = code for every entry of
   diffs[diff_offset[c] .. diff_offset[c+1]) (entry = stage << 16 | pos, code as a second word)
   and every offload bit flips[flip_offset[c] .. flip_offset[c+1]) toggled (bit = i*m + j). */
typedef struct ps_delta_batch {
    int64_t num_candidates;
    const uint16_t *ref_orders;     /* [P][order_stride]                                             */
    const uint32_t *ref_mask;       /* [mask_words]                                                  */
    const uint32_t *diff_offset;    /* [N+1], diff_offset[0] = 0                                     */
    const uint32_t *diffs;          /* [diff_offset[N]][2]: (stage << 16 | pos, code)                */
    const uint32_t *flip_offset;    /* [N+1]                                                         */
    const uint32_t *flips;          /* [flip_offset[N]] offload bit indices                          */
    const ps_base *base;            /* optional recorded base (as ps_cand_batch.base)                */
} ps_delta_batch;

/* Per-candidate outputs, device memory.  Optional arrays may be NULL. */
typedef struct ps_result_batch {
    int64_t *makespan;              /* [N] makespan in time quanta, -1 unless FEASIBLE             */
    double *bubble;                 /* [N] 1 - busy/(P*makespan) in fp64, NaN unless FEASIBLE      */
    int64_t *peak;                  /* [N][P] STRICT peak bytes per stage (optional)              */
    uint32_t *flags;                /* [N] PS_FLAG_*                                                */
    uint32_t *blocked;              /* [N] on DEADLOCK: bit i set = stage i still had ops (optional) */
    uint32_t *trace_code;           /* [N][trace_stride] commit-ordered events (optional)         */
    int32_t *trace_start;           /* [N][trace_stride] start times of those events (optional)   */
    int32_t trace_stride;           /* >= info.max_events when trace arrays are given             */
    int64_t *events_total;          /* device int64[2] (optional): [0] += events simulated (prefix /
                                       suffix sharing skips the rest), [1] += events the candidates
                                       have, 3Pm + 2 x offloaded (what a full evaluation commits) */
} ps_result_batch;

/* Local-search neighbourhood: how a candidate index becomes a move. */
typedef struct ps_move_params {
    uint64_t seed;
    uint32_t shift_permille;        /* share of SHIFT moves in 1/1000; the rest TOGGLE offload bits */
    uint32_t max_shift;             /* SHIFT distance drawn from 1..max_shift, either direction      */
} ps_move_params;

typedef struct ps_search_desc {
    const uint16_t *inc_orders;     /* device [P][order_stride]: incumbent structure — each stage
                                       row a permutation of its 3m ops (not re-validated per round;
                                       ps_eval_batch validates a structure, ps_apply_move keeps one) */
    const uint32_t *inc_mask;       /* device [mask_words]                                         */
    uint64_t round;
    int64_t first_index;            /* global index of this shard's first neighbour               */
    int64_t count;                  /* neighbours in this shard                                    */
    ps_move_params moves;
    int64_t *events_total;          /* device int64[2] (optional): as in ps_result_batch           */
    const ps_base *base;            /* optional: the incumbent recorded with ps_base_record        */
    int32_t dedup;                  /* 1 (with a base, no makespan_out): a move drawn several times
                                       in the round is simulated once, by its lowest index — the
                                       round's best key is the same                              */
    int64_t cutoff;                 /* > 0 (no makespan_out): the incumbent's makespan; a neighbour
                                       whose makespan provably reaches it (every stage's free time
                                       plus its remaining work) is abandoned — it
                                       cannot be a strict improvement, so the selection is the
                                       same.  0: every neighbour runs to its outcome.            */
} ps_search_desc;

/* A batch of branch-and-bound nodes (device buffers): the state solver._Search._bound reads. */
typedef struct ps_bound_batch {
    int64_t num_nodes;
    const int32_t *clock;           /* [N] node clock                                              */
    const int32_t *stage_free;      /* [N][P] stage free times                                     */
    const int32_t *comp_start;      /* [N][P][m][3] committed compute starts (F, B, W), -1 = not   */
} ps_bound_batch;

const char *ps_version(void);
const char *ps_last_error(void);

int ps_instance_create(const ps_instance_desc *desc, int device, ps_instance **out);
int ps_instance_destroy(ps_instance *inst);
int ps_instance_get_info(const ps_instance *inst, ps_instance_info *out);

/* Base recording for prefix sharing.  ps_base_record copies the candidate (device buffers
   [P][order_stride] and [mask_words]) and simulates it once, checkpointing as it goes; it returns
   after the recording (evaluations size their ledger window from what the base needed). */
int ps_base_create(const ps_instance *inst, ps_base **out);
int ps_base_destroy(ps_base *base);
int ps_base_record(ps_base *base, const uint16_t *orders, const uint32_t *mask, void *stream);
/* The same for a candidate with explicit channel orders (device [G][chan_stride], ps_cand_batch
   encoding): explicit-channel batches of that width (ps_eval_batch with channel_orders,
   ps_search_round_explicit with desc->base) then resume from its checkpoints and converge onto it,
   as derived-mode batches do with ps_base_record. */
int ps_base_record_explicit(ps_base *base, const uint16_t *orders, const uint32_t *mask,
                            const uint32_t *chan_orders, int32_t chan_stride, void *stream);
/* Inspection (tests, diagnostics): copy one recorded table to host memory after synchronising.
   what: PS_BASE_CHECKPOINTS [ck_max][ck_words] u32, PS_BASE_CSTEP [P][3m] u32, PS_BASE_FSTEP [P][m] u32,
   PS_BASE_INFO i32[8], PS_BASE_RESULT i64[2 + 3P], PS_BASE_LAYOUT i32[8] (ck_words, ck_max,
   ck_interval, window capacity, then the word offsets of the breakpoint times, their usages and the
   per-lane scalars inside a checkpoint, and the scalar words per lane).
   *bytes in: capacity, out: size of the table. */
enum { PS_BASE_CHECKPOINTS = 0, PS_BASE_CSTEP = 1, PS_BASE_FSTEP = 2, PS_BASE_INFO = 3, PS_BASE_RESULT = 4,
       PS_BASE_LAYOUT = 5 };
int ps_base_read(const ps_base *base, int what, void *host, size_t *bytes);

/* Lower bound of every node in the batch, one warp per node: replaces solver._Search._bound
   (solver.py:352-383) with _chain_ends (solver.py:321-350), bit-exact (int64 out, device [N]). */
int ps_bound_batch_eval(const ps_instance *inst, const ps_bound_batch *batch, int64_t *lower_bound, void *stream);

/* Evaluate N candidates (device buffers) on `stream` (a cudaStream_t, NULL = legacy default). */
int ps_eval_batch(const ps_instance *inst, const ps_cand_batch *batch,
                  const ps_result_batch *results, void *stream);

/* Same, with every pointer in batch/results in HOST memory (pinned for full copy speed).
   Synchronous: returns after results are back on the host. */
int ps_eval_batch_host(const ps_instance *inst, const ps_cand_batch *batch,
                       const ps_result_batch *results, void *stream);

/* ps_eval_batch_host on a delta-encoded batch (HOST buffers, results to HOST, synchronous): the
   differences cross PCIe and are classified on the device.  A candidate that is one move of the
   reference structure (one stage's contiguous run holding the reference run rotated by one, one
   offloadable bit flipped, or nothing) is evaluated by the move-encoded kernel against the
   reference (with prefix/suffix sharing when `base` was recorded on the reference); any other is
   rebuilt in HBM and evaluated materialised.  Derived channel mode.  Out-of-range entries or
   offsets fail the call (PS_ERR_INVALID) after the batch has run. */
int ps_eval_batch_host_delta(const ps_instance *inst, const ps_delta_batch *batch,
                             const ps_result_batch *results, void *stream);

/* One local-search round over neighbours [first_index, first_index+count) of the incumbent:
   generate each move, evaluate it, and atomically fold (makespan << 32 | index) of every
   feasible neighbour into *best_key (device int64, caller initialises it to INT64_MAX).
   makespan_out (device int64 [count], optional) receives every neighbour's makespan or -1. */
int ps_search_round(const ps_instance *inst, const ps_search_desc *desc,
                    int64_t *best_key, int64_t *makespan_out, void *stream);

/* The round of a search sharded over G ranks (one process per GPU): each rank
   passes its contiguous shard [first_index, first_index + count) of the round's global neighbour
   indices; after the local round the 8-byte key is combined across ranks with one
   ncclAllReduce(MIN) on `stream`, so every rank holds the round's global best key on return (the
   lowest global index wins ties, so the winner is the same for every G).  nccl_comm is an
   ncclComm_t owned by the caller (NULL = a single rank: the same as ps_search_round).
   libnccl.so.2 is loaded on first use (the library does not link against it).  Replaces the
   reference's sequential selection loop (heuristics.py:206; solver.py:437) for one round. */
int ps_search_round_sharded(const ps_instance *inst, const ps_search_desc *desc,
                            int64_t *best_key, int64_t *makespan_out, void *nccl_comm, void *stream);

/* The channel-order search: the incumbent carries explicit per-channel transfer
   orders inc_chan [G][chan_stride] (entries as in ps_cand_batch.channel_orders, padded with
   0xFFFFFFFF), replayed in explicit channel mode (listsched.py:233-239).  A neighbour is a
   stage-op shift (r0 % 1000 < shift_permille, or no transfers) or a shift of one transfer within
   its channel order — a reload (or offload) moved earlier or later among the channel's
   transfers (north star: "shift reloads").  Offload bits do not change.  Same key convention as
   ps_search_round; neighbours are materialised and evaluated as explicit-channel batches (no
   prefix sharing). */
int ps_search_round_explicit(const ps_instance *inst, const ps_search_desc *desc, const uint32_t *inc_chan,
                             int32_t chan_stride, int64_t *best_key, int64_t *makespan_out, void *stream);
/* Neighbours [first_index, first_index+count) as full candidates: orders [count][P][stride],
   masks [count][mask_words], channel orders [count][G][chan_stride] (device). */
int ps_materialize_moves_explicit(const ps_instance *inst, const ps_search_desc *desc, const uint32_t *inc_chan,
                                  int32_t chan_stride, uint16_t *orders_out, uint32_t *mask_out,
                                  uint32_t *chan_out, void *stream);
/* Apply neighbour `index` of `round` to the incumbent's stage and channel orders in place. */
int ps_apply_move_explicit(const ps_instance *inst, uint16_t *inc_orders, uint32_t *inc_chan, int32_t chan_stride,
                           const ps_move_params *moves, uint64_t round, uint64_t index, void *stream);

/* Materialise neighbours [first_index, first_index+count) as full candidates (device buffers
   shaped like ps_cand_batch: orders [count][P][order_stride], masks [count][mask_words]). */
int ps_materialize_moves(const ps_instance *inst, const ps_search_desc *desc,
                         uint16_t *orders_out, uint32_t *mask_out, void *stream);

/* Apply neighbour `index` of round `round` to the incumbent in place (device buffers). */
int ps_apply_move(const ps_instance *inst, uint16_t *inc_orders, uint32_t *inc_mask,
                  const ps_move_params *moves, uint64_t round, uint64_t index, void *stream);

/* INT32 issue-rate probe for the roofline denominator: runs `iters` dependent-free IADD3/LOP3
   chains on every SM; *lane_ops receives the lane-operations executed (device int64[1]). */
int ps_int32_probe(int64_t iters, int64_t *lane_ops, void *stream);

#ifdef __cplusplus
}
#endif

#endif /* PIPESCHED_B200_H */
