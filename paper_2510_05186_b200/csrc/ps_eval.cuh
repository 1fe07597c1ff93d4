// ps_eval.cuh — batched exact replica of the reference's earliest-feasible list scheduler.
//
// Reference semantics: listsched.run_order (listsched.py:167-269) commits,
// one event per step, the lexicographic minimum of (start, rank, OpId) over every stage head
// (compute, rank 0) and every transfer option (reload rank 1, offload rank 2), where
//   * a compute head's floor is its dependency floor (_compute_ready, listsched.py:114-145) and the
//     stage's free time; an F additionally waits for earliest_fit on its stage ledger with lag = T_F
//     (listsched.py:224-229);
//   * an offload's floor is its F's end, a reload's its offload's end, both clamped to the channel's
//     free time; a reload additionally waits for earliest_fit (listsched.py:186-204);
//   * commits put the compute delta at the op END, the offload's -G at its END and the reload's +G at
//     its START on the stage ledger (listsched.py:148-164).
//
// B200 mapping:
//   * one candidate per warp, one lane per stage (P <= 32): control flow is warp-uniform and the
//     argmin over stages is two REDUX.MIN over the 64-bit key (start:32 | rank:2 stage:6 mb:22 kind:2);
//   * every lane caches its stage's compute-head key and its best transfer key separately and
//     recomputes one only when the committed event can change its inputs (exact invalidation sets,
//     DESIGN.md §3.2), and caches earliest_fit answers until its ledger changes;
//   * the stage ledger is folded below a monotone line no future query or insertion can reach, so
//     only a short window of future points stays live; earliest_fit is a backward scan for the last
//     breakpoint whose usage exceeds limit - delta, exact;
//   * per-(stage, microbatch) end times are packed as (time << 2 | state) words in shared memory;
//   * a candidate whose window overflows is re-run by the GSTATE variant (state in global memory,
//     window = 5m, cannot overflow) from a device-side worklist — no host round trip, no CPU path.
#pragma once
#include <stdint.h>
#include <climits>
#include "ps_common.cuh"

namespace ps {

constexpr uint32_t FLAG_FEASIBLE = 1u, FLAG_DEADLOCK = 2u, FLAG_MALFORMED = 4u, FLAG_OVERFLOW = 8u,
                   FLAG_RANGE = 16u;   // an event time reached 2^29 quanta (see EvalParams::time_safe)
constexpr int TAU_NONE = INT_MAX;   // usage never drops far enough: earliest_fit returns None
constexpr int TAU_ANY = INT_MIN;    // fits at any query time at or above the fold line
constexpr uint32_t NO_CHAN = 0xFFFFFFFFu;

struct EvalParams {
    // instance (device tables)
    int P, m, G, L, MW, stride;
    int comm, toff, post, uniform, any_off;
    // Times are packed as (t << 2 | state) in 32 bits, so every event must END below 2^29: an event
    // chosen to start at or after time_safe = 2^29 - (longest duration) ends the candidate with
    // FLAG_RANGE.  INT_MAX when no schedule of the instance can get there (its horizon bound).
    int time_safe;
    int64_t busy, unit;
    const int32_t *proc;     // [rows][3]
    const void *vals;        // V [rows][4] = dF, dB, dW, gamma (in memory units)
    const void *limit;       // V [P]
    const int32_t *chan;     // [P]
    // materialised candidates
    int64_t N;
    const void *orders;      // uint16 op codes, or uint8 when order_u8
    int order_u8;
    const uint32_t *masks;
    const uint32_t *chorders;
    int chan_stride;
    // move-encoded candidates (search)
    const uint16_t *inc_orders;
    const uint32_t *inc_mask;
    uint64_t seed, round;
    int64_t first_index;
    uint32_t shift_permille, max_shift;
    const unsigned long long *move_list;   // explicit moves per candidate (pack_move), else Philox
    const int32_t *base_valid;             // optional device flag: 0 = the recorded base is not the
                                           // incumbent (no prefix sharing)
    // outputs
    int64_t *makespan;
    double *bubble;
    int64_t *peak;
    uint32_t *flags;
    uint32_t *blocked;
    uint32_t *tcode;
    int32_t *tstart;
    int tstride;
    long long *best_key;
    unsigned long long *events_total;   // optional: += committed events (roofline numerator)
    // overflow hand-off between the shared-memory and the global-state variant
    int32_t *ovf_list;
    int32_t *ovf_count;
    int32_t *work_next;      // dynamic candidate distribution (NULL: static grid stride)
    // streamed inputs (host-buffer evaluation): candidate c may be read once ready[c / ready_chunk]
    // is non-zero; the copy engine writes each flag after its chunk's data, on the same stream
    const int32_t *ready;
    long long ready_chunk;
    int dedup;               // (host side) evaluate each distinct move of a round once
    int win_smem;            // global-state passes: the ledger windows live in shared memory
    long long cutoff;        // > 0: abandon a neighbour whose makespan bound reaches it (§3.13)
    const int32_t *work_list;
    const int32_t *work_count;
    // per-candidate state
    int K;                   // ledger window capacity in merged breakpoints (2K slots per stage)
    int cand_words;          // 32-bit words of one candidate's state
    int inc_words;           // 32-bit words of the block-shared incumbent (move mode)
    uint32_t *gstate;        // GSTATE scratch
    // prefix sharing against a recorded base candidate
    int ck_interval;         // steps between checkpoints (power of two)
    int ck_words;            // words per checkpoint (layout independent of the window K, see below)
    int ck_kc;               // checkpoint window capacity per stage (the base was recorded with it)
    int ck_max;              // checkpoint capacity
    uint32_t *ck;            // [ck_max][ck_words]; NULL = no base
    uint32_t *cstep;         // [P][L] step at which the base commits stage i's q-th op (~0 = never)
    uint32_t *fstep;         // [P][m] step at which the base commits F(i, j)
    int32_t *base_info;      // [0] checkpoints (-1 unusable) [1] flags [2] events [3] blocked [4] max window
    int64_t *base_res;       // [0] makespan [1] bubble bits [2, 2+P) peaks [2+P, 2+2P) final free
                             // times [2+2P, 2+3P) first starts
    const uint16_t *base_orders;   // [P][stride] (materialised candidates; REC: the previous base)
    const uint32_t *base_mask;     // [mask_words]
    const uint32_t *base_chorders; // [G][chan_stride] explicit-channel base (REC: the previous base's)
    uint32_t *chstep;              // [G][chan_stride] compute events committed when the base commits
                                   // the transfer at that position of its channel order (~0 = never)
    int rec_prev;                  // REC: resume from the previous base's checkpoints
};

constexpr int CK_REGW = 24;          // per-lane register words saved in a checkpoint
constexpr uint32_t NEVER = 0xFFFFFFFFu;
// An A[i][j] word no future event reads (B(i,j), W(i,j) and B(i-1,j) all committed).  Dead words
// are canonical so that two simulations in the same live state compare equal.
constexpr uint32_t A_DEAD = 0xFFFFFFFFu;

template <typename V>
__device__ __forceinline__ V ldv(const void *base, int idx) {
    return __ldg(reinterpret_cast<const V *>(base) + idx);
}

// A candidate key: start in the high word, (rank, stage, microbatch, kind) in the low word.
// A warp's state words in 16-byte vectors: `dst`/`src` are 16-byte aligned (the host keeps the
// state block and every checkpoint on 4-word boundaries), the lanes stride over the vectors and
// the few words past the last whole vector.  Rolled: these run once per candidate, and the unrolled
// copies cost more in instruction fetch than they save.
__device__ __forceinline__ void warp_zero_words(uint32_t *dst, int n, int lane) {
    uint4 *d4 = reinterpret_cast<uint4 *>(dst);
    const int n4 = n >> 2;
#pragma unroll 1
    for (int k = lane; k < n4; k += 32) d4[k] = make_uint4(0u, 0u, 0u, 0u);
    for (int k = (n4 << 2) + lane; k < n; k += 32) dst[k] = 0u;
}
__device__ __forceinline__ void warp_copy_words(uint32_t *dst, const uint32_t *src, int n, int lane) {
    uint4 *d4 = reinterpret_cast<uint4 *>(dst);
    const uint4 *s4 = reinterpret_cast<const uint4 *>(src);
    const int n4 = n >> 2;
#pragma unroll 1
    for (int k = lane; k < n4; k += 32) d4[k] = s4[k];
    for (int k = (n4 << 2) + lane; k < n; k += 32) dst[k] = src[k];
}

// Global-state copies: U independent 16-byte loads in flight per lane before their stores (the
// rolled loop above exposes one L2 round trip per 512 bytes; config 5 restores 68 KB per neighbour).
template <int U>
__device__ __forceinline__ void warp_copy_words_mlp(uint32_t *dst, const uint32_t *src, int n, int lane) {
    uint4 *d4 = reinterpret_cast<uint4 *>(dst);
    const uint4 *s4 = reinterpret_cast<const uint4 *>(src);
    const int n4 = n >> 2;
    int k = lane;
#pragma unroll 1
    for (; k + 32 * (U - 1) < n4; k += 32 * U) {
        uint4 v[U];
#pragma unroll
        for (int u = 0; u < U; ++u) v[u] = s4[k + 32 * u];
#pragma unroll
        for (int u = 0; u < U; ++u) d4[k + 32 * u] = v[u];
    }
#pragma unroll 1
    for (; k < n4; k += 32) d4[k] = s4[k];
    for (int q = (n4 << 2) + lane; q < n; q += 32) dst[q] = src[q];
}

// Any-alignment warp copy/zero: 16-byte vectors when both ends allow, words otherwise.
__device__ __forceinline__ void warp_copy_words_any(uint32_t *dst, const uint32_t *src, int n, int lane) {
    if (((reinterpret_cast<uintptr_t>(dst) | reinterpret_cast<uintptr_t>(src)) & 15u) == 0) {
        warp_copy_words(dst, src, n, lane);
        return;
    }
#pragma unroll 1
    for (int k = lane; k < n; k += 32) dst[k] = src[k];
}
__device__ __forceinline__ void warp_zero_words_any(uint32_t *dst, int n, int lane) {
    if ((reinterpret_cast<uintptr_t>(dst) & 15u) == 0) {
        warp_zero_words(dst, n, lane);
        return;
    }
#pragma unroll 1
    for (int k = lane; k < n; k += 32) dst[k] = 0u;
}
// One lane's copy of words [lo, hi) of a row (band restore): with `vec`, the range
// widened to 16-byte boundaries (the caller guarantees the widened words are equal on both sides
// or irrelevant) and U vector loads in flight.
template <int U>
__device__ __forceinline__ void lane_copy_range(uint32_t *dst, const uint32_t *src, int lo, int hi, bool vec) {
    if (lo >= hi) return;
    if (vec) {
        uint4 *d4 = reinterpret_cast<uint4 *>(dst);
        const uint4 *s4 = reinterpret_cast<const uint4 *>(src);
        int k = lo >> 2;
        const int e = (hi + 3) >> 2;
#pragma unroll 1
        for (; k + U <= e; k += U) {
            uint4 v[U];
#pragma unroll
            for (int u = 0; u < U; ++u) v[u] = s4[k + u];
#pragma unroll
            for (int u = 0; u < U; ++u) d4[k + u] = v[u];
        }
#pragma unroll 1
        for (; k < e; ++k) d4[k] = s4[k];
        return;
    }
#pragma unroll 1
    for (int k = lo; k < hi; ++k) dst[k] = src[k];
}
__device__ __forceinline__ void lane_zero_range(uint32_t *dst, int lo, int hi, bool vec) {
    if (lo >= hi) return;
    if (vec) {
        uint4 *d4 = reinterpret_cast<uint4 *>(dst);
#pragma unroll 1
        for (int k = lo >> 2; k < (hi + 3) >> 2; ++k) d4[k] = make_uint4(0u, 0u, 0u, 0u);
        return;
    }
#pragma unroll 1
    for (int k = lo; k < hi; ++k) dst[k] = 0u;
}

__device__ __forceinline__ unsigned long long make_key(uint32_t hi, uint32_t lo) {
    return ((unsigned long long)hi << 32) | lo;
}
constexpr unsigned long long KEY_ABSENT = ~0ull;

// 72 registers per thread (7 blocks of 4 warps per SM) measured best on B200 for the
// shared-memory variants (tools/kvar.py: 64 spills the event loop's keys, 80+ loses warps);
// the global-state variant keeps its registers.
#ifndef PS_MIN_BLOCKS
#define PS_MIN_BLOCKS 7
#endif
// Data-dependent loops over ledger-window slots and state words stay rolled where the A/B says so:
// unrolled copies pushed the kernel past the instruction cache (ncu: no_instruction stalls 27%
// move-encoded, 45% materialised) and cost more in fetch than they saved in issue (r01 A/B,
// DESIGN.md §3.10).  PS_ROLL_HOT: event-loop window loops rolled 0 nowhere, 1 everywhere, 2 in the
// materialised-candidate kernels only (default: the move-encoded kernel gains from its unrolled
// copies on every config but the first rounds of config 3); PS_ROLL_COLD: the once-per-candidate ones.
#ifndef PS_ROLL_HOT
#define PS_ROLL_HOT 2
#endif
#ifndef PS_ROLL_COLD
#define PS_ROLL_COLD 1
#endif
#if PS_ROLL_HOT == 1
#define PS_HOT_LOOP(...) _Pragma("unroll 1") __VA_ARGS__
#elif PS_ROLL_HOT == 2          // rolled in the materialised-candidate kernels only
#define PS_HOT_LOOP(...) if constexpr (MOVES) { __VA_ARGS__ } else { _Pragma("unroll 1") __VA_ARGS__ }
#else
#define PS_HOT_LOOP(...) __VA_ARGS__
#endif
#if PS_ROLL_COLD
#define PS_NOUNROLL_C _Pragma("unroll 1")
#else
#define PS_NOUNROLL_C
#endif
#ifndef PS_GSTATE_MAX_WARPS
#define PS_GSTATE_MAX_WARPS 16 // global-memory state: warps per block sharing the incumbent copy
#endif
#ifndef PS_GSTATE_VEC_CMP
#define PS_GSTATE_VEC_CMP 0   // convergence-compare load schedule for global state: 1 = 16-byte loads, 2 = rows in flight
#endif
#ifndef PS_GSTATE_CMP_U
#define PS_GSTATE_CMP_U 4
#endif
#ifndef PS_GSTATE_COPY_MLP
#define PS_GSTATE_COPY_MLP 8  // global-state checkpoint restore: 16-byte loads in flight per lane (r01: 1 -> 8 is -7% config 5)
#endif
#ifndef PS_MIN_BLOCKS_G
#define PS_MIN_BLOCKS_G 1     // global-memory state: one 16-warp block per SM, 122 registers (r01 A/B)
#endif
#ifndef PS_MIN_BLOCKS_GNB
#define PS_MIN_BLOCKS_GNB 24  // global state without a base: one-warp blocks, <= 85 registers
#endif
#ifndef PS_MIN_BLOCKS_NB
#define PS_MIN_BLOCKS_NB 7    // materialised candidates without a base: full simulations (r02 A/B: 7 is -10% vs 5)
#endif
#ifndef PS_MIN_BLOCKS_MAT
#define PS_MIN_BLOCKS_MAT 5   // materialised candidates: 102-register cap (r01 A/B)
#endif
#ifndef PS_REC_BAND_CMP
#define PS_REC_BAND_CMP 1     // recordings compare row bands (per lane) rather than whole rows (warp-wide)
#endif
#ifndef PS_TAU_PAIR
#define PS_TAU_PAIR 0   // measured slower on B200 (r01): register pressure outweighs the saved scan
#endif

// DERIVED: greedy channel mode (no explicit channel orders); UNI: microbatch-symmetric tables.
// GS: per-candidate state in shared memory (0), in global scratch (1), in global scratch with
// nonzero-word masks over the pending-transfer sets (2: many bitset words per stage, config 5),
// in shared memory without a recorded base (3: materialised full simulations; no checkpoint code,
// built for 7 blocks per SM like the move-encoded kernel), in global scratch without a base (4:
// materialised full simulations of large shapes, one-warp blocks, PS_MIN_BLOCKS_GNB per SM).
template <typename V, bool MOVES, int GS, bool REC, bool DERIVED, bool UNI>
__global__ void __launch_bounds__((GS == 1 || GS == 2) ? 32 * PS_GSTATE_MAX_WARPS : GS == 4 ? 32 : 128,
                                  REC ? 1 : (GS == 1 || GS == 2) ? PS_MIN_BLOCKS_G : GS == 4 ? PS_MIN_BLOCKS_GNB
                                  : GS == 3 ? PS_MIN_BLOCKS_NB : (MOVES ? PS_MIN_BLOCKS : PS_MIN_BLOCKS_MAT))
eval_kernel(const EvalParams p) {
    constexpr bool GSTATE = GS == 1 || GS == 2 || GS == 4;
    constexpr bool NOBASE = GS == 3 || GS == 4;
    extern __shared__ __align__(16) uint32_t smem[];
    constexpr int VW = sizeof(V) / 4;
    const int lane = threadIdx.x & 31;
    const int warp = threadIdx.x >> 5;
    const int nwarps = blockDim.x >> 5;
    const int P = p.P, m = p.m, L = p.L, MW = p.MW, K = p.K;
    const int i = lane;                               // the stage this lane owns
    const bool has_stage = i < P;
    const int is = has_stage ? i : 0;
    constexpr bool derived = DERIVED;

    // ---- block-shared incumbent (move mode) ---------------------------------------------
    uint16_t *inc_s = reinterpret_cast<uint16_t *>(smem);
    uint32_t *incmask_s = smem + (P * p.stride + 1) / 2;
    if (MOVES) {
        const uint32_t *src = reinterpret_cast<const uint32_t *>(p.inc_orders);
        int nw = (P * p.stride) / 2;
        for (int k = threadIdx.x; k < nw; k += blockDim.x) smem[k] = src[k];
        for (int k = threadIdx.x; k < (P * m + 31) / 32; k += blockDim.x) incmask_s[k] = p.inc_mask[k];
        __syncthreads();
    }

    // ---- this warp's state slot ----------------------------------------------------------
    const long long slot = (long long)blockIdx.x * nwarps + warp;
    const long long nslots = (long long)gridDim.x * nwarps;
    // State words are addressed as 32-bit offsets from the shared-memory symbol (or from the
    // warp's global scratch slot): no 64-bit pointers stay live across the event loop.
    uint32_t *const gsw = GSTATE ? p.gstate + (size_t)slot * p.cand_words : nullptr;
    const int sbase = p.inc_words + warp * p.cand_words;       // shared-memory word offset
#define SW(off) (GSTATE ? gsw[(off)] : smem[sbase + (off)])
#define SV(off) (GSTATE ? reinterpret_cast<V *>(gsw)[(off)] : reinterpret_cast<V *>(smem)[sbase / VW + (off)])
    const int o_wu = is * 2 * K;                                // own ledger window: usage after (V units)
    const int o_wt = P * 2 * K * VW + is * 2 * K;               // own ledger window: times
    const int o_A = P * 2 * K * (VW + 1);                       // [P][m] F end, then B end (time<<2 | state)
    const int o_Ai = o_A + is * m;
    const int o_Xi = o_A + P * m + is * m;                      // [P][m] offload end, then reload end
    // Per-stage bitsets [3][P][MW] (offloaded, pending offloads, pending reloads), addressed by SB()
    // relative to their start: after the rows in the state block, or (global-state passes) in the
    // warp's slice of shared memory behind the incumbent, where the event loop's many reads of them
    // stay on chip (checkpoints keep them after the rows either way).
    const int o_bits = GSTATE ? 0 : o_A + 2 * P * m;           // bitsets' start, in SB() offsets
    const int o_offm = o_bits + is * MW;                        // [P][MW] offloaded bits
    const int o_poff = o_offm + P * MW;                         // [P][MW] pending offload requests
    const int o_prel = o_poff + P * MW;                         // [P][MW] pending reload requests
    const int nb3 = 3 * P * MW;                                 // bitset words
    const int nz = 2 * P * m + nb3;                      // words zeroed per candidate
    const int sbits = p.inc_words + warp * ((nb3 + 3) & ~3);    // (global state) shared-memory bitsets
#define SB(off) (GSTATE ? smem[sbits + (off)] : smem[sbase + (off)])
    // Ledger windows (offsets o_wu / o_wt from the state start): with win_smem, a global-state pass
    // keeps them in the warp's shared-memory slice behind all warps' bitsets (same layout).
    uint32_t *const wsw = !GSTATE ? nullptr
                        : p.win_smem ? smem + p.inc_words + nwarps * ((nb3 + 3) & ~3) + warp * (P * 2 * K * (VW + 1))
                                     : gsw;
#define SWW(off) (GSTATE ? wsw[(off)] : smem[sbase + (off)])
#define SVW(off) (GSTATE ? reinterpret_cast<V *>(wsw)[(off)] : reinterpret_cast<V *>(smem)[sbase / VW + (off)])
    // materialised candidates: the candidate's stage orders, staged once (16-byte aligned: row8
    // reads eight uint16 codes at a time; the state start and o_A are 16-byte aligned)
    const int o_row = o_A + ((nz + 3) & ~3);
    const int row_bytes = P * p.stride * (p.order_u8 ? 1 : 2);

    const int chan_i = has_stage ? __ldg(&p.chan[i]) : -1;
    // this stage's host link is its own (no other stage transfers on it)
    const bool chan_excl = __popc(__match_any_sync(0xffffffffu, chan_i)) == 1;
    const V limit_i = has_stage ? ldv<V>(p.limit, i) : V(0);
    const int rowbase = UNI ? is : is * m;
    // per-stage constants of microbatch-symmetric instances live in registers
    int t0 = 0, t1 = 0, t2 = 0;
    V v0 = 0, v1 = 0, v2 = 0, v3 = 0;
    if (UNI) {
        t0 = __ldg(&p.proc[rowbase * 3 + 0]);
        t1 = __ldg(&p.proc[rowbase * 3 + 1]);
        t2 = __ldg(&p.proc[rowbase * 3 + 2]);
        v0 = ldv<V>(p.vals, rowbase * 4 + 0);
        v1 = ldv<V>(p.vals, rowbase * 4 + 1);
        v2 = ldv<V>(p.vals, rowbase * 4 + 2);
        v3 = ldv<V>(p.vals, rowbase * 4 + 3);
    }
    auto proc_of = [&](int j, int k) -> int {
        if (UNI) return k == 0 ? t0 : (k == 1 ? t1 : t2);
        return __ldg(&p.proc[(rowbase + j) * 3 + k]);
    };
    auto val_of = [&](int j, int k) -> V {
        if (UNI) return k == 0 ? v0 : (k == 1 ? v1 : (k == 2 ? v2 : v3));
        return ldv<V>(p.vals, (rowbase + j) * 4 + k);
    };

    // ---- per-lane registers ----------------------------------------------------------------
    long long cand = 0;
    Move mv;
    mv.type = MOVE_NOOP; mv.stage = 0; mv.a = mv.b = 0; mv.mb = 0;
    int pos = 0, sfree = 0, cfree = 0;
    unsigned long long ckey = KEY_ABSENT;      // cached compute-head key
    unsigned long long tkey = KEY_ABSENT;      // cached best transfer key of this stage
    bool cdirty = false, tdirty = false, ovf = false;
    V base = 0, top = 0, peak = 0;
    V segpk = 0;                               // REC: max usage folded since the last checkpoint
    int ws = 0, we = 0;
    int wlo = INT_MAX, whi = INT_MIN;          // times of the window's first / last breakpoint
    int n_poff = 0, n_prel = 0, n_unrel = 0;   // pending offloads / reloads / offloaded not yet reloaded
    // earliest_fit cache, valid until the ledger changes; NO_R marks it empty (R >= -delta > NO_R)
    constexpr V NO_R = (V)(sizeof(V) == 8 ? (V)0x8000000000000000LL : (V)0x80000000);
    V rF = NO_R, rG = NO_R;
    int tauF = 0, tauG = 0;
    int first_start = INT_MAX;      // start of the stage's first op (always an F; its last op is always a W)
    int rem = 0;                    // (bound pruning) work of this stage's uncommitted ops
    int ecount = 0, ecount0 = 0;             // events committed / restored from a checkpoint
    int cc = 0;                              // compute events committed (checkpoints count these)
    uint32_t head = 0, nxt = 0;
    int cpos = 0;
    uint32_t chead = NO_CHAN, cnext = NO_CHAN;
    int wt = -1;        // see compute_key
    int lastq = -1;     // last position of this stage's order that differs from the base's
    int lastqc = -1;    // explicit channels: last position of this lane's channel order that differs
    int eoff = 0;       // base step = candidate step + eoff once the candidate's extra/missing transfers are done
    // Row bands.  A stage's end-time rows are A_DEAD (A row) / zero (X row) below the
    // band of microbatches in flight and zero above it, in the slot as in every checkpoint (whose band
    // a recording saves in register word 21/22).  Global-state evaluation passes (BAND) therefore
    // restore and compare only the rows' bands: this lane's A row is A_DEAD below b_alo, its X row
    // zero below b_xlo, both zero from b_hi on (the slot starts unknown: everything is rewritten).
    // A recording tracks the same bounds to save them.
    constexpr bool BAND = GSTATE && !REC;
    // Global state: which words of this stage's pending-offload (bits 0-15) and pending-reload
    // (bits 16-31) sets are nonzero, so transfer_key skips the empty ones (config 5: 8 words each).
    const bool wmask_on = GS == 2 && MW <= 16;     // (GS 2 is launched for 6 <= MW <= 16 only)
    uint32_t pwm = 0;
    int b_alo = 0, b_xlo = 0, b_hi = m;
    // 16-byte vectors over the rows: row starts and checkpoints on 16-byte boundaries
    const bool band_vec = ((o_A | m | p.cand_words | p.ck_words) & 3) == 0;

    // op code idx of the staged candidate rows ([P][stride], uint8 or uint16)
    auto row_at = [&](int idx) -> uint32_t {
        const unsigned char *rb = GSTATE ? reinterpret_cast<const unsigned char *>(gsw + o_row)
                                         : reinterpret_cast<const unsigned char *>(smem + sbase + o_row);
        return p.order_u8 ? (uint32_t)rb[idx] : (uint32_t)reinterpret_cast<const uint16_t *>(rb)[idx];
    };
    // eight op codes from position q (a multiple of 8) of stage i's staged row, as uint16 pairs
    auto row8 = [&](int q) -> uint4 {
        const unsigned char *rb = GSTATE ? reinterpret_cast<const unsigned char *>(gsw + o_row)
                                         : reinterpret_cast<const unsigned char *>(smem + sbase + o_row);
        if (!p.order_u8) return *reinterpret_cast<const uint4 *>(rb + 2 * (i * p.stride + q));
        const uint2 b = *reinterpret_cast<const uint2 *>(rb + i * p.stride + q);
        return make_uint4(__byte_perm(b.x, 0u, 0x4140), __byte_perm(b.x, 0u, 0x4342),
                          __byte_perm(b.y, 0u, 0x4140), __byte_perm(b.y, 0u, 0x4342));
    };
    auto fetch = [&](int q) -> uint32_t {
        if (q >= L || !has_stage) return 0u;
        if (MOVES) {
            int src = (mv.type == MOVE_SHIFT && i == mv.stage) ? shifted_position(q, mv.a, mv.b) : q;
            return inc_s[i * p.stride + src];
        }
        return row_at(i * p.stride + q);
    };
    auto fetch_chan = [&](int q) -> uint32_t {
        if (derived || !has_stage || q >= p.chan_stride) return NO_CHAN;
        return __ldg(&p.chorders[((size_t)cand * p.G + chan_i) * p.chan_stride + q]);
    };

    // The recorded base's offload bits of this stage, re-based to [MW] words (the incumbent's in
    // move mode: the base is always the incumbent there).
    auto base_word = [&](int w) -> uint32_t {
        const int mwords = (P * m + 31) / 32;
        const int gb = i * m + w * 32, q = gb >> 5, sh = gb & 31;
        auto word = [&](int qq) -> uint32_t {
            if (qq >= mwords) return 0u;
            return MOVES ? incmask_s[qq] : __ldg(&p.base_mask[qq]);
        };
        uint32_t bits = word(q) >> sh;
        if (sh) bits |= word(q + 1) << (32 - sh);
        const int nb = m - w * 32;
        if (nb < 32) bits &= (1u << nb) - 1u;
        return bits;
    };

    // Ledger window: the stage's merged breakpoints at or after the fold line, sorted by time, each
    // holding the usage AFTER it; slots [ws, we) of a 2K array, compacted when the end is reached.
    // base = usage at the fold line (the last folded breakpoint's), top = usage after everything.
    auto win_fold = [&](int line) {
        PS_HOT_LOOP(while (ws < we && wlo < line) {
            V u = SVW(o_wu + (ws));
            peak = u > peak ? u : peak;
            if (REC) segpk = u > segpk ? u : segpk;
            base = u;
            ++ws;
            wlo = ws < we ? (int)SWW(o_wt + (ws)) : INT_MAX;
        })
        if (ws == we) whi = INT_MIN;
    };
    // Called before sfree / cfree / n_unrel reflect the event being committed: the fold line is
    // below sfree, and below the channel's free time while this stage still has a transfer to come,
    // so no future query or insertion (this one included) lands under it.
    auto win_insert = [&](int t, V d) {
        // (greedy channels: with no transfer of this stage in flight, every later transfer of it
        // follows an F not committed yet, so nothing can land below the stage free time)
        win_fold((derived ? (n_poff > 0 || n_prel > 0) : n_unrel > 0) ? min(sfree, cfree) : sfree);
        top += d;
        rF = rG = NO_R;                                // the ledger changed: drop cached answers
        int k = we - 1;
        if (ws < we && t == whi) {                     // same time as the last breakpoint: merge
            SVW(o_wu + (k)) += d;
            return;
        }
        if (ws < we && t < whi) {
            PS_HOT_LOOP(while (k >= ws && (int)SWW(o_wt + (k)) > t) --k;)  // last breakpoint at or before t
            if (k >= ws && (int)SWW(o_wt + (k)) == t) {          // same time: merge into that breakpoint
                PS_HOT_LOOP(for (int q = k; q < we; ++q) SVW(o_wu + (q)) += d;)
                return;
            }
        }
        if (we - ws == K) { ovf = true; return; }
        if (we == 2 * K) {                             // compact to the front
            PS_HOT_LOOP(for (int q = ws; q < we; ++q) { SWW(o_wt + (q - ws)) = SWW(o_wt + (q)); SVW(o_wu + (q - ws)) = SVW(o_wu + (q)); })
            k -= ws;
            we -= ws;
            ws = 0;
        }
        PS_HOT_LOOP(for (int q = we - 1; q > k; --q) { SWW(o_wt + (q + 1)) = SWW(o_wt + (q)); SVW(o_wu + (q + 1)) = SVW(o_wu + (q)) + d; })
        SWW(o_wt + (k + 1)) = (uint32_t)t;
        SVW(o_wu + (k + 1)) = (k >= ws ? SVW(o_wu + (k)) : base) + d;
        ++we;
        if (k + 1 == we - 1) whi = t;                  // appended
        if (k + 1 == ws) wlo = t;                      // new first breakpoint
    };
    // earliest_fit core: first breakpoint after the last one whose usage exceeds R.
    auto win_tau = [&](V R) -> int {
        if (R < 0 || top > R) return TAU_NONE;
        int k = we - 1;
        PS_HOT_LOOP(while (k >= ws && !(SVW(o_wu + (k)) > R)) --k;)
        if (k >= ws) return (int)SWW(o_wt + (k + 1));
        return base > R && ws < we ? (int)SWW(o_wt + (ws)) : TAU_ANY;
    };
    // Symmetric tables: the F and reload thresholds are per-stage constants with R_G >= R_F, so one
    // backward scan finds the last breakpoint above R_F and, continuing, the last above R_G.
    auto tau_pair = [&]() {
        const V RF = limit_i - v0, RG = limit_i - v3;
        int k = we - 1;
        PS_HOT_LOOP(while (k >= ws && !(SVW(o_wu + (k)) > RF)) --k;)
        const int kF = k;
        PS_HOT_LOOP(while (k >= ws && !(SVW(o_wu + (k)) > RG)) --k;)
        auto conv = [&](V R, int kk) -> int {
            if (R < 0 || top > R) return TAU_NONE;
            if (kk >= ws) return (int)SWW(o_wt + (kk + 1));
            return base > R && ws < we ? (int)SWW(o_wt + (ws)) : TAU_ANY;
        };
        tauF = conv(RF, kF);
        tauG = conv(RG, k);
        rF = RF;
        rG = RG;
    };
    auto tau_F = [&](V R) -> int {
        if (R != rF) {
            if (UNI && PS_TAU_PAIR) tau_pair();
            else { tauF = win_tau(R); rF = R; }
        }
        return tauF;
    };
    auto tau_G = [&](V R) -> int {
        if (R != rG) {
            if (UNI && PS_TAU_PAIR) tau_pair();
            else { tauG = win_tau(R); rG = R; }
        }
        return tauG;
    };

    // wt: the stage whose uncommitted op the head waits for (-1: none, or memory / a transfer)
    auto compute_key = [&]() {
        ckey = KEY_ABSENT;
        wt = -1;
        if (!has_stage || pos >= L) return;
        const int j = head >> 2, k = head & 3u;
        int fl;
        if (k == KIND_F) {
            fl = 0;
            if (i > 0) {
                uint32_t a = SW(o_A + ((i - 1) * m + j));
                if (!(a & 3u)) { wt = i - 1; return; }
                fl = (int)(a >> 2) + p.comm;
            }
        } else if (k == KIND_B) {
            uint32_t a = SW(o_Ai + (j));
            if ((a & 3u) != 1u) { wt = i; return; }      // F(i, j) comes later in this stage's order
            fl = (int)(a >> 2);
            if (i < P - 1) {
                uint32_t b = SW(o_A + ((i + 1) * m + j));
                if ((b & 3u) < 2u) { wt = i + 1; return; }   // 2: B committed, 3: and W too
                fl = max(fl, (int)(b >> 2) + p.comm);
            }
            if ((SB(o_offm + (j >> 5)) >> (j & 31)) & 1u) {
                uint32_t x = SW(o_Xi + (j));
                if ((x & 3u) != 2u) return;
                fl = max(fl, (int)(x >> 2));
            }
        } else {
            uint32_t a = SW(o_Ai + (j));
            if ((a & 3u) != 2u) { wt = i; return; }      // B(i, j) comes later in this stage's order
            fl = (int)(a >> 2);
        }
        int lo = max(fl, sfree);
        if (k == KIND_F) {
            int tau = tau_F(limit_i - val_of(j, 0));
            if (tau == TAU_NONE) {
                // the usage after everything committed stays too high; only this stage's pending
                // offloads could lower it before the head commits (B/W are behind it): none left
                // means waiting for itself
                if (derived && n_poff == 0) wt = i;
                return;
            }
            if (tau != TAU_ANY) lo = max(lo, tau - proc_of(j, 0));
        }
        ckey = make_key((uint32_t)lo, ((uint32_t)i << 24) | ((uint32_t)j << 2) | (uint32_t)k);
    };

    auto transfer_key = [&]() {
        unsigned long long best = KEY_ABSENT;
        const int C = cfree;
        const uint32_t stb = (uint32_t)i << 24;
        if (derived) {
            // (global state: only the words the nonzero-word masks name)
            auto poff_word = [&](int w) {
                for (uint32_t bits = SB(o_poff + (w)); bits; bits &= bits - 1) {
                    int j = w * 32 + __ffs(bits) - 1;
                    best = min(best, make_key((uint32_t)max((int)(SW(o_Ai + (j)) >> 2), C),
                                              (2u << 30) | stb | ((uint32_t)j << 2)));
                }
            };
            auto prel_word = [&](int w) {
                for (uint32_t bits = SB(o_prel + (w)); bits; bits &= bits - 1) {
                    int j = w * 32 + __ffs(bits) - 1;
                    int tau = tau_G(limit_i - val_of(j, 3));
                    if (tau == TAU_NONE) continue;
                    best = min(best, make_key((uint32_t)max(max((int)(SW(o_Xi + (j)) >> 2), C), tau),
                                              (1u << 30) | stb | ((uint32_t)j << 2)));
                }
            };
            if (n_poff) {
                if (wmask_on) for (uint32_t x = pwm & 0xFFFFu; x; x &= x - 1) poff_word(__ffs(x) - 1);
                else for (int w = 0; w < MW; ++w) poff_word(w);
            }
            if (n_prel) {
                if (wmask_on) for (uint32_t x = pwm >> 16; x; x &= x - 1) prel_word(__ffs(x) - 1);
                else for (int w = 0; w < MW; ++w) prel_word(w);
            }
        } else if (chead != NO_CHAN && (int)((chead >> 16) & 0x7FFFu) == i) {
            int j = chead & 0xFFFFu;
            if (!(chead >> 31)) {
                uint32_t a = SW(o_Ai + (j));
                if (a & 3u) best = make_key((uint32_t)max((int)(a >> 2), C), (2u << 30) | stb | ((uint32_t)j << 2));
            } else {
                uint32_t x = SW(o_Xi + (j));
                if ((x & 3u) == 1u) {
                    int tau = tau_G(limit_i - val_of(j, 3));
                    if (tau != TAU_NONE) {
                        best = make_key((uint32_t)max(max((int)(x >> 2), C), tau), (1u << 30) | stb | ((uint32_t)j << 2));
                    }
                }
            }
        }
        tkey = best;
    };

    // Lane 0 publishes a candidate's outcome (search rounds may pass no arrays).
    // full_ev: the candidate's algorithmic event count 3Pm + 2|off| (roofline numerator, credited
    // to feasible outcomes); a deadlocked candidate is credited only with the events the reference
    // commits before it raises, of which `dl_ev` (committed here, or by the base it matched) is a
    // lower bound.
    int full_ev = 0;
    auto put_result = [&](uint32_t flag, long long span, uint32_t blocked_mask, int dl_ev) {
        if (p.events_total && ecount > ecount0) atomicAdd(p.events_total, (unsigned long long)(ecount - ecount0));
        if (p.events_total && (flag & (FLAG_FEASIBLE | FLAG_DEADLOCK)))
            atomicAdd(p.events_total + 1, (unsigned long long)(flag == FLAG_FEASIBLE ? full_ev : max(dl_ev, 0)));
        if (p.flags) p.flags[cand] = flag;
        if (p.makespan) p.makespan[cand] = span;
        if (p.bubble)
            p.bubble[cand] = span > 0 ? 1.0 - (double)p.busy / ((double)P * (double)span)
                                      : __longlong_as_double(0x7ff8000000000000LL);
        if (p.blocked) p.blocked[cand] = blocked_mask;
#ifdef PS_DEBUG_EVENTS
        // diagnostics build: simulated events | restored-from step << 16 in place of the bubble
        // (tools/event_stats.py; early deadlock detection stays on without a blocked output)
        if (p.bubble) p.bubble[cand] = (double)((uint32_t)(ecount - ecount0) | ((uint32_t)min(ecount0, 32767) << 16));
#endif
    };

    // Checkpoint c: the state before the base commits its compute event number c*C (compute
    // events, not all events: a candidate with other offload bits runs other transfers but the
    // same 3Pm computes, so its states line up with the base's).  Independent of the evaluating
    // pass's window K:
    //   [0, nz)               A, X, offm, poff, prel
    //   [ck_t, ck_t + P*KC)   each stage's live breakpoint times, compacted to slot 0
    //   [ck_u, ck_u + P*KC*VW) their usages
    //   [ck_r, ck_r + 32*CK_REGW) every lane's scalars (window as ws = 0, we = count): 0-8 see
    //                         save_regs, 9 widest window so far, 10-11 peak folded since the
    //                         previous checkpoint, 12-17 base/top/peak, 18-19 peak folded after
    //                         this checkpoint (S_c), 20 event step
    const int ck_t = (nz + 1) & ~1;
    const int ck_u = (ck_t + P * p.ck_kc + 1) & ~1;
    const int ck_r = ck_u + P * p.ck_kc * VW;
    auto save_regs = [&](uint32_t *rg) {
        rg[0] = pos; rg[1] = sfree; rg[2] = cfree; rg[3] = ws; rg[4] = we; rg[5] = n_poff; rg[6] = n_prel;
        rg[7] = n_unrel; rg[8] = first_start;
        rg[23] = (uint32_t)cpos;                 // explicit channels: this lane's channel cursor
        *reinterpret_cast<long long *>(rg + 12) = (long long)base;
        *reinterpret_cast<long long *>(rg + 14) = (long long)top;
        *reinterpret_cast<long long *>(rg + 16) = (long long)peak;
    };
    auto load_regs = [&](const uint32_t *rg) {
        pos = rg[0]; sfree = rg[1]; cfree = rg[2]; ws = rg[3]; we = rg[4]; n_poff = rg[5]; n_prel = rg[6];
        n_unrel = rg[7]; first_start = rg[8];
        if (!derived) cpos = (int)rg[23];
        base = (V)*reinterpret_cast<const long long *>(rg + 12);
        top = (V)*reinterpret_cast<const long long *>(rg + 14);
        peak = (V)*reinterpret_cast<const long long *>(rg + 16);
    };
    const int n_ck = (!NOBASE && p.ck && !REC && (!p.base_valid || *p.base_valid)) ? p.base_info[0] : 0;
    // Checkpoints to resume from: the base's for a candidate; for a re-recording (REC with
    // rec_prev) those of the previous base, whose prefix the new one shares up to their divergence.
    const int n_src = REC ? (p.rec_prev ? p.base_info[0] : 0) : n_ck;

    // Suffix sharing: every offload bit on which the candidate and the base differ
    // is dead once that microbatch's B has committed on this stage.
    auto diff_dead = [&]() -> bool {
        for (int w = 0; w < MW; ++w)
            for (uint32_t x = SB(o_offm + (w)) ^ base_word(w); x; x &= x - 1)
                if ((SW(o_Ai + (w * 32 + __ffs(x) - 1)) & 3u) < 2u) return false;
        return true;
    };
    // The time below which end-time word k (value w) is irrelevant: a pending reader on another
    // resource waits for that resource's free time, which only grows, so a time at or below it
    // (minus the comm lag) can never matter again.  INT_MAX-free: INT_MAX = no such reader.
    // Warp-collective (shuffles): every lane calls it; `need` selects the lanes that use it.
    auto dom_bound = [&](bool need, int k, uint32_t w) -> int {
        const bool isA = k < P * m;
        const int kk = isA ? k : k - P * m;
        const int si = need ? kk / m : 0, j = need ? kk - si * m : 0;
        const int sf_up = __shfl_sync(0xffffffffu, sfree, min(si + 1, 31));
        const int sf_dn = __shfl_sync(0xffffffffu, sfree, max(si - 1, 0));
        const int sf_own = __shfl_sync(0xffffffffu, sfree, si);
        const int cf_own = __shfl_sync(0xffffffffu, cfree, si);
        int bound = INT_MAX;
        if (need) {
            const uint32_t st = w & 3u;
            if (isA && st == 1u) {          // F end: F(si+1, j), and F(si, j)'s offload
                if (si + 1 < P && (SW(o_A + ((si + 1) * m + j)) & 3u) == 0u) bound = min(bound, sf_up - p.comm);
                if (((SB(o_bits + si * MW + (j >> 5)) >> (j & 31)) & 1u) &&
                    (SW(o_A + (P * m + si * m + j)) & 3u) == 0u)
                    bound = min(bound, cf_own);
            } else if (isA) {               // B end: B(si-1, j)
                if (si > 0 && (SW(o_A + ((si - 1) * m + j)) & 3u) < 2u) bound = min(bound, sf_dn - p.comm);
            } else if (st == 2u) {          // reload end: B(si, j)
                bound = min(bound, sf_own);
            }
        }
        return bound;
    };
    // Recording: drop every such time at each checkpoint boundary, so checkpoints hold only times
    // that still matter (simulations are unchanged; state bits are untouched, so the predicates
    // other lanes read meanwhile are stable).
    // dom_bound for a word of this lane's own rows (j: microbatch, st: its state), given the
    // neighbouring stages' free times: no shuffles, for per-lane loops over the row bands.
    auto own_bound = [&](bool isA, int j, uint32_t st, int sf_up, int sf_dn) -> int {
        int bound = INT_MAX;
        if (isA && st == 1u) {
            if (i + 1 < P && (SW(o_A + ((i + 1) * m + j)) & 3u) == 0u) bound = min(bound, sf_up - p.comm);
            if (((SB(o_offm + (j >> 5)) >> (j & 31)) & 1u) && (SW(o_Xi + (j)) & 3u) == 0u) bound = min(bound, cfree);
        } else if (isA) {
            if (i > 0 && (SW(o_A + ((i - 1) * m + j)) & 3u) < 2u) bound = min(bound, sf_dn - p.comm);
        } else if (st == 2u) {
            bound = min(bound, sfree);
        }
        return bound;
    };
    auto canon_dominated = [&]() {
        // each lane over its own rows' band (outside it no word carries a time)
        const int sf_up = __shfl_sync(0xffffffffu, sfree, min(i + 1, 31));
        const int sf_dn = __shfl_sync(0xffffffffu, sfree, max(i - 1, 0));
        if (has_stage) {
            while (b_alo < b_hi && SW(o_Ai + (b_alo)) == A_DEAD) ++b_alo;
            auto canon = [&](bool isA, int j, uint32_t w) -> uint32_t {
                if ((w >> 2) == 0u || w == A_DEAD) return w;
                const int bound = own_bound(isA, j, w & 3u, sf_up, sf_dn);
                return bound != INT_MAX && (int)(w >> 2) <= bound ? (w & 3u) : w;
            };
            for (int r = 0; r < 2; ++r) {
                const int off = r == 0 ? o_Ai : o_Xi;
                if (band_vec) {
                    // four words per 16-byte access (the widened words are A_DEAD or zero: unchanged)
                    uint4 *row4 = reinterpret_cast<uint4 *>(&SW(off));
#pragma unroll 1
                    for (int k = b_alo >> 2; k < (b_hi + 3) >> 2; ++k) {
                        const uint4 v = row4[k];
                        const uint4 c = make_uint4(canon(r == 0, 4 * k, v.x), canon(r == 0, 4 * k + 1, v.y),
                                                   canon(r == 0, 4 * k + 2, v.z), canon(r == 0, 4 * k + 3, v.w));
                        if (c.x != v.x || c.y != v.y || c.z != v.z || c.w != v.w) row4[k] = c;
                    }
                } else {
#pragma unroll 1
                    for (int j = b_alo; j < b_hi; ++j) SW(off + (j)) = canon(r == 0, j, SW(off + (j)));
                }
            }
        }
        __syncwarp();
    };
    // Is this candidate's live state before its current step that of the base before step c*C,
    // up to one time shift `delta` of every live time (stage and channel free times, live F/B and
    // transfer end times, ledger breakpoints; usages, positions and pending sets equal)?  The
    // scheduler is translation invariant on such states — every start is a max of live times plus
    // constants, every commit adds a constant, the fold line moves with them — so the candidate
    // continues as the base does, `delta` later.
    bool rec_chg = false;        // REC: this stage's offload bits differ from the previous base's
    int rec_dn = 0;              // REC: and its count of offloaded activations by this much
    // A recording's suffix peaks: walking c from `hi` down to 0, rg[18] of checkpoint c = run, then
    // run = max(run, rg[10]) (the peak folded in c's interval); eight loads in flight per batch.
    auto suffix_peaks = [&](int hi, long long run) {
        constexpr int U = 8;
        int c = hi;
        for (; c - (U - 1) >= 0; c -= U) {
            long long sg[U];
#pragma unroll
            for (int u = 0; u < U; ++u)
                sg[u] = *reinterpret_cast<const long long *>(p.ck + (size_t)(c - u) * p.ck_words + ck_r + lane * CK_REGW + 10);
#pragma unroll
            for (int u = 0; u < U; ++u) {
                *reinterpret_cast<long long *>(p.ck + (size_t)(c - u) * p.ck_words + ck_r + lane * CK_REGW + 18) = run;
                run = sg[u] > run ? sg[u] : run;
            }
        }
        for (; c >= 0; --c) {
            uint32_t *rg = p.ck + (size_t)c * p.ck_words + ck_r + lane * CK_REGW;
            const long long sg = *reinterpret_cast<const long long *>(rg + 10);
            *reinterpret_cast<long long *>(rg + 18) = run;
            run = sg > run ? sg : run;
        }
    };
    int conv_delta = 0;
    auto same_state = [&](int c) -> bool {
        const uint32_t *src = p.ck + (size_t)c * p.ck_words;
        const uint32_t *rg = src + ck_r + lane * CK_REGW;
        bool eq = true;
        const int d = __shfl_sync(0xffffffffu, sfree - (int)rg[1], 0);
        // the per-stage scalars first: they tell a still-perturbed candidate apart cheaply
        if (has_stage) {
            // a channel that has carried nothing yet (free time 0 on both) constrains nothing
            // (nor does an own channel with nothing in flight that is already behind the stage: every
            // later transfer on it waits for an F not committed yet)
            eq = pos == (int)rg[0] && sfree - (int)rg[1] == d && (derived || cpos == (int)rg[23]) &&
                 (cfree - (int)rg[2] == d || (cfree == 0 && rg[2] == 0u) ||
                  (derived && chan_excl && n_poff == 0 && n_prel == 0 && cfree <= sfree && rg[2] <= rg[1])) &&
                 we - ws == (int)rg[4] &&
                 n_poff == (int)rg[5] && n_prel == (int)rg[6] && n_unrel == (int)rg[7] &&
                 (first_start == INT_MAX) == ((int)rg[8] == INT_MAX) &&
                 (long long)base == *reinterpret_cast<const long long *>(rg + 12) &&
                 (long long)top == *reinterpret_cast<const long long *>(rg + 14);
        }
#ifdef PS_DEBUG_CONV
        // diagnostics build: histogram of the first failing component into events_total[2 + r]
        auto dbg = [&](int r) { if (lane == 0 && p.events_total) atomicAdd(p.events_total + 2 + r, 1ull); };
        {
            int r = 99;
            if (has_stage) {
                if (pos != (int)rg[0]) r = 0;
                else if (sfree - (int)rg[1] != d) r = 1;
                else if (!(cfree - (int)rg[2] == d || (cfree == 0 && rg[2] == 0u))) r = 2;
                else if (we - ws != (int)rg[4]) r = 3;
                else if (n_poff != (int)rg[5] || n_prel != (int)rg[6] || n_unrel != (int)rg[7]) r = 4;
                else if ((first_start == INT_MAX) != ((int)rg[8] == INT_MAX)) r = 5;
                else if ((long long)base != *reinterpret_cast<const long long *>(rg + 12) ||
                         (long long)top != *reinterpret_cast<const long long *>(rg + 14)) r = 6;
            }
            r = __reduce_min_sync(0xffffffffu, r);
            if (r != 99) dbg(r);
            // would exempting finished stages (pos == L in both) from the time/window checks pass?
            int r2 = 99;
            if (has_stage && !(pos == L && (int)rg[0] == L)) {
                if (pos != (int)rg[0]) r2 = 0;
                else if (sfree - (int)rg[1] != d) r2 = 1;
                else if (!(cfree - (int)rg[2] == d || (cfree == 0 && rg[2] == 0u))) r2 = 2;
                else if (we - ws != (int)rg[4]) r2 = 3;
            }
            r2 = __reduce_min_sync(0xffffffffu, r2);
            if (r != 99 && r2 == 99) dbg(10);
        }
#endif
        if (!__all_sync(0xffffffffu, eq)) return false;
        // end-time words (time << 2 | state): a time the base's checkpoint still carries (it
        // matters there) must be the candidate's moved by delta; a time the checkpoint dropped must
        // be irrelevant in the candidate too (dom_bound); state-only words must be equal
        const uint32_t d4 = (uint32_t)d << 2;
        const int n2 = 2 * P * m;
        if constexpr (BAND || (REC && PS_REC_BAND_CMP)) {
            // Each lane compares its own stage's rows over the union of the two bands (outside it
            // both sides are A_DEAD below and zero above), 16-byte vectors, two of each in flight.
            // dom_bound's readers are this stage's neighbours: their free times are shuffled once.
            const int sf_up = __shfl_sync(0xffffffffu, sfree, min(i + 1, 31));
            const int sf_dn = __shfl_sync(0xffffffffu, sfree, max(i - 1, 0));
            if (has_stage) {
                while (b_alo < b_hi && SW(o_Ai + (b_alo)) == A_DEAD) ++b_alo;   // (monotone: amortised)
                b_xlo = max(b_xlo, b_alo);                                    // A_DEAD => X word zero
                const int hi = max(b_hi, (int)rg[22]);
                auto word_ok = [&](bool isA, int j, uint32_t cw, uint32_t bw) -> bool {
                    const bool timed_c = (cw >> 2) != 0u && cw != A_DEAD, timed_b = (bw >> 2) != 0u && bw != A_DEAD;
                    if (timed_c == timed_b && (timed_c ? cw - bw == d4 : cw == bw)) return true;
                    if (!(timed_c && !timed_b && (cw & 3u) == bw)) return false;
                    const int bound = own_bound(isA, j, cw & 3u, sf_up, sf_dn);
                    return bound != INT_MAX && (int)(cw >> 2) <= bound;
                };
                auto cmp_row = [&](bool isA, int row_off, const uint32_t *brow, int lo) -> bool {
                    if (lo >= hi) return true;
                    if (band_vec) {
                        const uint4 *c4 = reinterpret_cast<const uint4 *>(&SW(row_off));
                        const uint4 *b4 = reinterpret_cast<const uint4 *>(brow);
                        const int e = (hi + 3) >> 2;
#pragma unroll 1
                        for (int k = lo >> 2; k < e; k += 2) {
                            const bool two = k + 1 < e;
                            const uint4 ca = c4[k], ba = b4[k];
                            const uint4 cb = two ? c4[k + 1] : ca, bb = two ? b4[k + 1] : ba;
                            const int j = 4 * k;
                            if (!(word_ok(isA, j, ca.x, ba.x) && word_ok(isA, j + 1, ca.y, ba.y) &&
                                  word_ok(isA, j + 2, ca.z, ba.z) && word_ok(isA, j + 3, ca.w, ba.w)))
                                return false;
                            if (two && !(word_ok(isA, j + 4, cb.x, bb.x) && word_ok(isA, j + 5, cb.y, bb.y) &&
                                         word_ok(isA, j + 6, cb.z, bb.z) && word_ok(isA, j + 7, cb.w, bb.w)))
                                return false;
                        }
                        return true;
                    }
#pragma unroll 1
                    for (int j = lo; j < hi; ++j)
                        if (!word_ok(isA, j, SW(row_off + j), brow[j])) return false;
                    return true;
                };
                const int clo = (int)rg[21];
                eq = cmp_row(true, o_Ai, src + i * m, min(b_alo, clo)) &&
                     cmp_row(false, o_Xi, src + P * m + i * m, min(b_xlo, clo));
            }
        } else if (GSTATE && PS_GSTATE_VEC_CMP == 2) {
            // same test, PS_GSTATE_CMP_U coalesced rows of loads in flight before they are tested
            constexpr int U = PS_GSTATE_CMP_U;
            for (int k0 = 0; k0 < n2; k0 += 32 * U) {
                uint32_t cws[U], bws[U];
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    const int k = k0 + 32 * u + lane;
                    cws[u] = k < n2 ? SW(o_A + (k)) : 0u;
                    bws[u] = k < n2 ? src[k] : 0u;
                }
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    const uint32_t cw = cws[u], bw = bws[u];
                    const bool timed_c = (cw >> 2) != 0u && cw != A_DEAD, timed_b = (bw >> 2) != 0u && bw != A_DEAD;
                    bool ok = (timed_c == timed_b) && (timed_c ? cw - bw == d4 : cw == bw);
                    const bool relax = !ok && timed_c && !timed_b && (cw & 3u) == bw;
                    if (__any_sync(0xffffffffu, relax)) {
                        const int bound = dom_bound(relax, k0 + 32 * u + lane, cw);
                        if (relax) ok = bound != INT_MAX && (int)(cw >> 2) <= bound;
                    }
                    eq = eq && ok;
                }
            }
        } else if (GSTATE && PS_GSTATE_VEC_CMP == 1) {
            // same test, four words per lane per 16-byte load (state and checkpoint are 16-byte aligned)
            for (int k0 = 0; k0 < n2; k0 += 128) {
                const int kb = k0 + 4 * lane;
                uint32_t cws[4], bws[4];
                if (kb + 3 < n2) {
                    const uint4 c4 = *reinterpret_cast<const uint4 *>(&SW(o_A + (kb)));
                    const uint4 b4 = *reinterpret_cast<const uint4 *>(src + kb);
                    cws[0] = c4.x; cws[1] = c4.y; cws[2] = c4.z; cws[3] = c4.w;
                    bws[0] = b4.x; bws[1] = b4.y; bws[2] = b4.z; bws[3] = b4.w;
                } else {
#pragma unroll
                    for (int q = 0; q < 4; ++q) {
                        cws[q] = kb + q < n2 ? SW(o_A + (kb + q)) : 0u;
                        bws[q] = kb + q < n2 ? src[kb + q] : 0u;
                    }
                }
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    const uint32_t cw = cws[q], bw = bws[q];
                    const bool timed_c = (cw >> 2) != 0u && cw != A_DEAD, timed_b = (bw >> 2) != 0u && bw != A_DEAD;
                    bool ok = (timed_c == timed_b) && (timed_c ? cw - bw == d4 : cw == bw);
                    const bool relax = !ok && timed_c && !timed_b && (cw & 3u) == bw;
                    if (__any_sync(0xffffffffu, relax)) {
                        const int bound = dom_bound(relax, kb + q, cw);
                        if (relax) ok = bound != INT_MAX && (int)(cw >> 2) <= bound;
                    }
                    eq = eq && ok;
                }
                if ((k0 & 1023) == 896 && !__all_sync(0xffffffffu, eq)) return false;
            }
        } else
        for (int k0 = 0; k0 < n2; k0 += 32) {
            const int k = k0 + lane;
            uint32_t cw = 0u, bw = 0u;
            if (k < n2) { cw = SW(o_A + (k)); bw = src[k]; }
            const bool timed_c = (cw >> 2) != 0u && cw != A_DEAD, timed_b = (bw >> 2) != 0u && bw != A_DEAD;
            bool ok = (timed_c == timed_b) && (timed_c ? cw - bw == d4 : cw == bw);
            const bool relax = !ok && timed_c && !timed_b && (cw & 3u) == bw;
            if (__any_sync(0xffffffffu, relax)) {
                const int bound = dom_bound(relax, k, cw);
                if (relax) ok = bound != INT_MAX && (int)(cw >> 2) <= bound;
            }
            eq = eq && ok;
        }
#ifdef PS_DEBUG_CONV
        if (!__all_sync(0xffffffffu, eq)) { dbg(7); return false; }
#endif
        PS_NOUNROLL_C for (int k = P * MW + lane; k < nb3; k += 32)     // (offm skipped: its differences are dead)
            eq = eq && SB(o_bits + k) == src[2 * P * m + k];
#ifdef PS_DEBUG_CONV
        if (!__all_sync(0xffffffffu, eq)) { dbg(8); return false; }
#endif
        if (has_stage && eq) {
            const uint32_t *st = src + ck_t + i * p.ck_kc;
            const V *su = reinterpret_cast<const V *>(src + ck_u) + i * p.ck_kc;
            PS_NOUNROLL_C for (int q = 0; q < we - ws && eq; ++q)
                eq = (int)SWW(o_wt + (ws + q)) - (int)st[q] == d && SVW(o_wu + (ws + q)) == su[q];
        }
        conv_delta = d;
#ifdef PS_DEBUG_CONV
        if (!__all_sync(0xffffffffu, eq)) dbg(9); else dbg(11);
#endif
        return __all_sync(0xffffffffu, eq);
    };

    const long long n_items = p.work_list ? (long long)*p.work_count : p.N;
    // Candidates cost from tens to thousands of events: after the first, each warp takes the next
    // unclaimed one (one atomic per candidate) so no SM idles behind a few long simulations.
    long long item = slot;
    auto next_item = [&]() -> long long {
        if (!p.work_next) return item + nslots;
        int v = 0;
        if (lane == 0) v = atomicAdd(p.work_next, 1);
        return nslots + (long long)__shfl_sync(0xffffffffu, v, 0);
    };
    for (; item < n_items; item = next_item()) {
        cand = p.work_list ? (long long)p.work_list[item] : item;
        if (p.ready) {
            // this candidate's chunk may still be crossing PCIe: wait for its flag
            if (lane == 0) {
                const volatile int32_t *f = p.ready + cand / p.ready_chunk;
                // (bounded: a flag that never comes — a failed copy — aborts the launch, ~10 s)
                for (unsigned spins = 0; *f == 0; ++spins) {
                    if (spins > (1u << 25)) __trap();
                    __nanosleep(256);
                }
                __threadfence();
            }
            __syncwarp();
        }
        // ================= initialise ======================================================
        // (BAND: the rows are rewritten over their bands by the restore below; only the bitsets here)
        if (BAND) warp_zero_words_any(&SB(o_bits), nb3, lane);
        else warp_zero_words(&SW(o_A), nz, lane);
        if (!MOVES) {
            // stage the candidate's rows: 8-byte loads, coalesced across the warp
            const uint2 *src = reinterpret_cast<const uint2 *>(reinterpret_cast<const unsigned char *>(p.orders) +
                                                               (size_t)cand * row_bytes);
            uint2 *dst = GSTATE ? reinterpret_cast<uint2 *>(gsw + o_row) : reinterpret_cast<uint2 *>(smem + sbase + o_row);
            for (int k = lane; k < row_bytes / 8; k += 32) dst[k] = __ldcg(src + k);   // (L2: may be streamed in)
        }
        if (MOVES) {
            uint64_t gidx = (uint64_t)(p.first_index + cand);
            if (p.move_list) {
                mv = unpack_move(p.move_list[cand]);
                if (mv.type >= MOVE_GENERAL) {          // (warp-uniform) evaluated by another pass
                    __syncwarp();
                    continue;
                }
            } else {
                mv = decode_move(p.seed, p.round, gidx, P, m, p.shift_permille, p.max_shift, p.any_off != 0,
                                 [&](int s, int j) { return ldv<V>(p.vals, (UNI ? s : s * m + j) * 4 + 3) > V(0); });
            }
        }
        __syncwarp();
        bool bad = false;
        // this stage's offload bits of the candidate, re-based to [MW] words; returns their count
        auto build_mask = [&](bool check) -> int {
            const int mwords = (P * m + 31) / 32;
            int n = 0;
            for (int w = 0; w < MW; ++w) {
                // bits [i*m + 32w, i*m + 32w + 32) of the packed candidate mask
                const int gb = i * m + w * 32, q = gb >> 5, sh = gb & 31;
                auto word = [&](int qq) -> uint32_t {
                    if (qq >= mwords) return 0u;
                    return MOVES ? incmask_s[qq] : __ldcg(&p.masks[(size_t)cand * mwords + qq]);
                };
                uint32_t bits = word(q) >> sh;
                if (sh) bits |= word(q + 1) << (32 - sh);
                const int nb = m - w * 32;
                if (nb < 32) bits &= (1u << nb) - 1u;
                if (MOVES && mv.type == MOVE_TOGGLE && mv.stage == i && (mv.mb >> 5) == w) bits ^= 1u << (mv.mb & 31);
                SB(o_offm + (w)) = bits;
                n += __popc(bits);
                // an offload bit on a non-offloadable op is malformed (KeyError in the reference)
                if (check)
                    for (uint32_t t = bits; t; t &= t - 1)
                        if (!(val_of(w * 32 + __ffs(t) - 1, 3) > 0)) bad = true;
            }
            return n;
        };
        int cand_unrel = 0;
        lastq = -1;
        lastqc = -1;
        int dq = L;         // first position where the row differs from the recorded base's
        if (has_stage) {
            cand_unrel = build_mask(true);
            if (!MOVES) {
                bool full = true;
                if (n_src > 0) {
                    // first and last position where the row differs from the (well-formed) base's,
                    // eight codes at a time (rows are padded to a multiple of 8)
                    const uint16_t *brow = p.base_orders + (size_t)i * p.stride;
                    auto differs8 = [&](int q) -> bool {
                        const uint4 a = row8(q), b = __ldg(reinterpret_cast<const uint4 *>(brow + q));
                        return a.x != b.x || a.y != b.y || a.z != b.z || a.w != b.w;
                    };
                    int q = 0;
                    while (q + 8 <= L && !differs8(q)) q += 8;
                    while (q < L && row_at(i * p.stride + q) == brow[q]) ++q;
                    dq = q;
                    if (q < L) {
                        int e = L - 1;          // every position above e is equal
                        while (e > q && ((e + 1) & 7) && row_at(i * p.stride + e) == brow[e]) --e;
                        if (((e + 1) & 7) == 0)
                            while (e - 7 > q && !differs8(e - 7)) e -= 8;
                        while (e > q && row_at(i * p.stride + e) == brow[e]) --e;
                        lastq = e;
                    }
                    // equal to a permutation outside [dq, lastq]: a permutation iff that window holds
                    // the base window's codes, each once
                    if (dq == L) {
                        full = false;
                    } else if (lastq - dq < 16) {
                        full = false;
                        for (int t = dq; t <= lastq && !bad; ++t) {
                            const uint32_t c = row_at(i * p.stride + t);
                            bool found = false;
                            for (int u = dq; u <= lastq; ++u) found = found || brow[u] == c;
                            for (int u = dq; u < t; ++u) bad = bad || row_at(i * p.stride + u) == c;
                            bad = bad || !found;
                        }
                    }
                }
                // otherwise the whole order must be a permutation of the stage's 3m ops: 3m valid
                // codes without a repeat (seen-sets in registers up to m = 64, else in the A row)
                if (!full) {
                } else if (m <= 64) {
                    unsigned long long fm = 0ull, bm = 0ull, wm = 0ull;
                    for (int q = 0; q < L; ++q) {
                        const uint32_t op = row_at(i * p.stride + q), j = op >> 2, k = op & 3u;
                        if (j >= (uint32_t)m || k > 2u) { bad = true; break; }
                        const unsigned long long bit = 1ull << j;
                        const unsigned long long seen = k == 0u ? fm : (k == 1u ? bm : wm);
                        if (seen & bit) { bad = true; break; }
                        if (k == 0u) fm |= bit; else if (k == 1u) bm |= bit; else wm |= bit;
                    }
                } else {
                    if (BAND) {            // the row is the seen-set scratch: clear it first
                        lane_zero_range(&SW(o_Ai), 0, b_hi, band_vec);
                        b_alo = 0;
                    }
                    for (int q = 0; q < L; ++q) {
                        uint32_t op = row_at(i * p.stride + q);
                        uint32_t j = op >> 2, k = op & 3u;
                        if (j >= (uint32_t)m || k > 2u || (SW(o_Ai + (j)) >> k) & 1u) { bad = true; break; }
                        SW(o_Ai + (j)) |= 1u << k;
                    }
                    for (int j = 0; j < m; ++j) SW(o_Ai + (j)) = 0u;
                }
            }
        }
        if (!MOVES && !derived && lane < p.G) {
            // explicit channel orders name offloaded activations of stages on their channel (the
            // literal replay decides what the reference does with anything else)
            const uint32_t *crow = p.chorders + ((size_t)cand * p.G + lane) * p.chan_stride;
            const int mwords = (P * m + 31) / 32;
            for (int q = 0; q < p.chan_stride && !bad; ++q) {
                const uint32_t e = __ldg(crow + q);
                if (e == NO_CHAN) break;
                const int s2 = (int)((e >> 16) & 0x7FFFu), j2 = (int)(e & 0xFFFFu);
                if (s2 >= P || j2 >= m || __ldg(&p.chan[s2]) != lane) { bad = true; break; }
                const int bit = s2 * m + j2;
                if (!((__ldcg(&p.masks[(size_t)cand * mwords + (bit >> 5)]) >> (bit & 31)) & 1u)) bad = true;
            }
        }
        if (__any_sync(0xffffffffu, bad)) {
            if (lane == 0) put_result(FLAG_MALFORMED, -1LL, 0u, 0);
            if (REC && lane == 0) {
                // a malformed base is unusable (and must not leave the previous one's tables live)
                p.base_info[0] = -1;
                p.base_info[1] = (int)FLAG_MALFORMED;
                p.base_info[5] = -1;
            }
            __syncwarp();
            continue;
        }
        if (p.events_total) {
            // the candidate's own event count: 3Pm computes and two transfers per offloaded F
            const int n_off = __reduce_add_sync(0xffffffffu, has_stage ? cand_unrel : 0);
            full_ev = 3 * P * m + 2 * n_off;
        }
        // ---- prefix sharing: the first step whose inputs differ from the recorded base ----
        uint32_t div = 0u;
        eoff = 0;
        if (n_src > 0) {
            uint32_t d = NEVER;
            if (has_stage) {
                // the base's last compute event before which stage i's head is still position q
                auto after = [&](int q) -> uint32_t { return q == 0 ? 0u : p.cstep[i * L + q - 1]; };
                int nbase = 0;
                if (MOVES) {
                    if (mv.stage == i) {
                        if (mv.type == MOVE_SHIFT) { d = after(min(mv.a, mv.b)); lastq = max(mv.a, mv.b); }
                        else if (mv.type == MOVE_TOGGLE) d = p.fstep[i * m + mv.mb];
                    }
                    for (int w = 0; w < MW; ++w) nbase += __popc(base_word(w));
                } else {
                    if (dq < L) d = after(dq);       // (dq, lastq: found while validating)
                    for (int w = 0; w < MW; ++w) {
                        const uint32_t bb = base_word(w);
                        nbase += __popc(bb);
                        for (uint32_t x = SB(o_offm + (w)) ^ bb; x; x &= x - 1)
                            d = min(d, p.fstep[i * m + w * 32 + __ffs(x) - 1]);
                    }
                }
                eoff = nbase - cand_unrel;
            }
            if (!derived) {
                // explicit channel orders: lane g compares channel g's order with the base's; the
                // first difference at position q takes effect once the base has committed the
                // transfer at q - 1 (checkpoints before the compute event preceding it are safe)
                int lq = -1;
                if (lane < p.G) {
                    const uint32_t *crow = p.chorders + ((size_t)cand * p.G + lane) * p.chan_stride;
                    const uint32_t *brow = p.base_chorders + (size_t)lane * p.chan_stride;
                    int qc = 0;
                    while (qc < p.chan_stride && crow[qc] == brow[qc]) ++qc;
                    if (qc < p.chan_stride) {
                        int e = p.chan_stride - 1;
                        while (e > qc && crow[e] == brow[e]) --e;
                        lq = e;
                        uint32_t dc = 0u;
                        if (qc > 0) {
                            const uint32_t y = p.chstep[(size_t)lane * p.chan_stride + qc - 1];
                            dc = y == NEVER ? NEVER : (y > 0u ? y - 1u : 0u);
                        }
                        d = min(d, dc);
                    }
                }
                lastqc = __shfl_sync(0xffffffffu, lq, chan_i >= 0 ? chan_i : 0);
            }
            // the base runs two transfer events per offloaded activation the candidate does not have
            eoff = 2 * __reduce_add_sync(0xffffffffu, eoff);
            div = __reduce_min_sync(0xffffffffu, d);
            if (REC && div == NEVER) div = 0u;        // same base again: record it afresh
            if (div == NEVER) {
                // identical to the base up to its end: its outcome is this candidate's
                if (p.peak && has_stage) p.peak[(size_t)cand * P + i] = p.base_res[2 + i];
                if (lane == 0) {
                    ecount = ecount0 = 0;
                    const long long span = p.base_res[0];
                    put_result((uint32_t)p.base_info[1], span, (uint32_t)p.base_info[3], p.base_info[2]);
                    if (MOVES && p.best_key && span >= 0) {
                        long long key = (span << 32) | (long long)(uint32_t)(p.first_index + cand);
                        if (key < *(volatile long long *)p.best_key) atomicMin(p.best_key, key);
                    }
                }
                __syncwarp();
                continue;
            }
        }
        const int ck_idx = n_src > 0 ? min((int)(div / (uint32_t)p.ck_interval), n_src - 1) : 0;
        if (ck_idx > 0) {
            const uint32_t *src = p.ck + (size_t)ck_idx * p.ck_words;
            load_regs(src + ck_r + lane * CK_REGW);
            if (__any_sync(0xffffffffu, has_stage && we > K)) {
                // the base's window at this point does not fit this pass: hand over to a wider pass
                if (lane == 0 && p.ovf_list) {
                    int at = atomicAdd(p.ovf_count, 1);
                    p.ovf_list[at] = (int32_t)cand;
                }
                __syncwarp();
                continue;
            }
#if PS_SYNC_ARGMIN
            __syncwarp();      // every lane's writes of its stage's offload bits before the restore's
#endif
            if (BAND) {
                // the bitsets, then each stage's rows over the old and the checkpoint's band
                warp_copy_words_any(&SB(o_bits), src + 2 * P * m, nb3, lane);
                if (has_stage) {
                    const uint32_t *rgs = src + ck_r + lane * CK_REGW;
                    const int clo = (int)rgs[21], chi = (int)rgs[22];
                    const int hi = max(b_hi, chi);
                    lane_copy_range<4>(&SW(o_Ai), src + i * m, min(b_alo, clo), hi, band_vec);
                    lane_copy_range<4>(&SW(o_Xi), src + P * m + i * m, min(b_xlo, clo), hi, band_vec);
                    b_alo = b_xlo = clo;
                    b_hi = chi;
                }
            } else if (GSTATE) {
                warp_copy_words_mlp<PS_GSTATE_COPY_MLP>(&SW(o_A), src, nz, lane);
            } else {
                warp_copy_words(&SW(o_A), src, nz, lane);
            }
            if (REC && has_stage) {
                b_alo = b_xlo = (int)src[ck_r + lane * CK_REGW + 21];
                b_hi = (int)src[ck_r + lane * CK_REGW + 22];
            }
            if (has_stage) {
                const uint32_t *st = src + ck_t + i * p.ck_kc;
                const V *su = reinterpret_cast<const V *>(src + ck_u) + i * p.ck_kc;
                PS_NOUNROLL_C for (int q = 0; q < we; ++q) { SWW(o_wt + (q)) = st[q]; SVW(o_wu + (q)) = su[q]; }
                wlo = we > 0 ? (int)st[0] : INT_MAX;
                whi = we > 0 ? (int)st[we - 1] : INT_MIN;
            }
            __syncwarp();
            if (has_stage) {
                // this candidate's offload bits: any difference lies on an F the base has not
                // committed yet, so only the outstanding-transfer count moves
                int nb = 0;
                for (int w = 0; w < MW; ++w) nb += __popc(SB(o_offm + (w)));
                n_unrel += cand_unrel - nb;
                if (REC) {
                    // did this stage's offload bits change from the previous base's (restored above)?
                    bool chg = false;
                    for (int w = 0; w < MW; ++w) {
                        const int gb = i * m + w * 32, q = gb >> 5, sh = gb & 31, mwords = (P * m + 31) / 32;
                        uint32_t bits = (q < mwords ? __ldcg(&p.masks[(size_t)cand * mwords + q]) : 0u) >> sh;
                        if (sh && q + 1 < mwords) bits |= __ldcg(&p.masks[(size_t)cand * mwords + q + 1]) << (32 - sh);
                        const int nbits = m - w * 32;
                        if (nbits < 32) bits &= (1u << nbits) - 1u;
                        chg = chg || bits != SB(o_offm + (w));
                    }
                    rec_chg = chg;
                    rec_dn = cand_unrel - nb;
                }
                build_mask(false);
                if (wmask_on) {
                    pwm = 0;
                    for (int w = 0; w < MW; ++w)
                        pwm |= (SB(o_poff + (w)) ? 1u << w : 0u) | (SB(o_prel + (w)) ? 1u << (16 + w) : 0u);
                }
            }
            if (REC) {
                // The kept checkpoints become the new base's: its offload bits, and the
                // outstanding-transfer count that goes with them (the suffix-sharing compare reads
                // both) — only for the stages whose bits changed (none after a shift), with the
                // lanes striding over the checkpoints so their loads overlap.
                const int dn = has_stage ? rec_dn : 0;
                __syncwarp();
                for (unsigned chg = __ballot_sync(0xffffffffu, has_stage && rec_chg); chg; chg &= chg - 1) {
                    const int st = __ffs(chg) - 1;
                    const int dns = __shfl_sync(0xffffffffu, dn, st);
                    for (int c = lane; c <= ck_idx; c += 32) {
                        uint32_t *dst = p.ck + (size_t)c * p.ck_words;
                        for (int w = 0; w < MW; ++w) dst[2 * P * m + st * MW + w] = SB(o_bits + st * MW + w);
                        if (dns) dst[ck_r + st * CK_REGW + 7] += (uint32_t)dns;
                    }
                }
            }
            ecount = (int)src[ck_r + 20];               // (lane 0's copy: warp-uniform by construction)
            ecount0 = ecount;
            cc = ck_idx * p.ck_interval;
        } else {
            if (BAND && has_stage) {
                lane_zero_range(&SW(o_Ai), 0, b_hi, band_vec);
                lane_zero_range(&SW(o_Xi), b_xlo, b_hi, band_vec);
            }
            b_alo = b_xlo = b_hi = 0;
            ecount0 = 0;
            pos = 0; sfree = 0; cfree = 0;
            base = top = peak = 0; ws = we = 0;
            wlo = INT_MAX; whi = INT_MIN;
            n_poff = n_prel = 0;
            pwm = 0;
            n_unrel = cand_unrel;
            first_start = INT_MAX; ecount = 0;
            cc = 0;
        }
        // Bound pruning (search rounds with a cutoff): the stage's remaining work
        const bool prune = MOVES && !REC && p.cutoff > 0;
        if (prune) {
            rem = 0;
            if (has_stage)
                for (int q = pos; q < L; ++q) {
                    const uint32_t op = fetch(q);
                    rem += proc_of((int)(op >> 2), (int)(op & 3u));
                }
        }
        bool pruned = false;
        const int cc0 = cc;
        ovf = false;
        rF = rG = NO_R;
        head = fetch(pos); nxt = fetch(pos + 1);
        if (ck_idx <= 0) cpos = 0;                   // (a restored candidate resumes its channel cursor)
        chead = fetch_chan(cpos); cnext = fetch_chan(cpos + 1);
        cdirty = tdirty = has_stage;
        ckey = tkey = KEY_ABSENT;
        __syncwarp();

        // ================= simulate: one committed event per iteration ===================
        bool ck_full = false;
        // a resumed recording starts from the previous base's widest window up to its checkpoint
        int max_win = REC && cc0 > 0 ? (int)p.ck[(size_t)(cc0 / p.ck_interval) * p.ck_words + ck_r + 9] : 0;
        int conv_c = -1;
        bool early_dl = false;
        bool range_ovf = false;
        for (;;) {
            if (REC) max_win = max(max_win, __reduce_max_sync(0xffffffffu, we - ws));
            if (cdirty) { compute_key(); cdirty = false; }
            if (!REC && !p.blocked && (ecount & 3) == 0) {
                // Early deadlock: a stage whose head waits for an op behind itself in its own order,
                // or two neighbours whose heads wait for each other, can never move again, so the
                // run ends in OrderInfeasible.  Only the set of stages left would still change, and
                // no output here reports it.  (Checked every 4th event: a wait, once permanent,
                // stays so.)
                const int nx = __shfl_sync(0xffffffffu, wt, min(i + 1, 31));
                const bool stuck = wt == i || (wt == i + 1 && nx == i);      // (wt >= 0: no key)
                if (__any_sync(0xffffffffu, stuck)) { early_dl = true; break; }
                if (prune) {
                    // every remaining op of a stage runs after its free time: the makespan is at
                    // least max(free + remaining work) - min(first start) (per-stage spans under
                    // post-validation); no strict improvement once that reaches the incumbent's
                    long long lb;
                    if (p.post) {
                        lb = __reduce_max_sync(0xffffffffu, has_stage && first_start != INT_MAX
                                                                ? (unsigned)(sfree + rem - first_start) : 0u);
                    } else {
                        const int hi = (int)__reduce_max_sync(0xffffffffu, has_stage ? (unsigned)(sfree + rem) : 0u);
                        const int lo = (int)__reduce_min_sync(0xffffffffu, has_stage ? (unsigned)first_start : 0x7FFFFFFFu);
                        lb = (long long)hi - (long long)lo;
                    }
                    if (lb >= p.cutoff) { pruned = true; break; }
                }
            }
            if (tdirty) { transfer_key(); tdirty = false; }
            const unsigned long long key = min(ckey, tkey);
            const uint32_t kh = (uint32_t)(key >> 32);
            const uint32_t mh = __reduce_min_sync(0xffffffffu, kh);
            const uint32_t ml = __reduce_min_sync(0xffffffffu, kh == mh ? (uint32_t)key : 0xFFFFFFFFu);
            if (mh == KEY_NONE) break;

            const int t = (int)mh;
            if (t >= p.time_safe) { range_ovf = true; break; }     // (warp-uniform)
            const int rank = (int)(ml >> 30);
            if (rank == RANK_COMPUTE && (cc & (p.ck_interval - 1)) == 0) {
                const int c = cc / p.ck_interval;
                // Suffix sharing.  A re-recording converges onto the previous base the same way:
                // it saves this checkpoint, then stops, and the remaining ones are the previous
                // base's shifted (rec_shift_kernel).
                if (REC) canon_dominated();
                if ((REC ? n_src > 1 : n_ck > 1) && cc > (int)div && c < n_src) {
                    const bool gate = !ovf && (!has_stage || (pos > lastq && diff_dead() && (derived || cpos > lastqc)));
                    if (__all_sync(0xffffffffu, gate)) {
                        if (same_state(c)) {
                            conv_c = c;
                            if (!REC) break;
                        }
                    }
                }
                // (a re-recording keeps the previous base's checkpoint it resumed from: same state)
                if (REC && !(cc == cc0 && cc0 > 0)) {
                    if (c < p.ck_max) {
                        uint32_t *dst = p.ck + (size_t)c * p.ck_words;
                        warp_copy_words(dst, &SW(o_A), nz, lane);
                        if (has_stage) {
                            uint32_t *st = dst + ck_t + i * p.ck_kc;
                            V *su = reinterpret_cast<V *>(dst + ck_u) + i * p.ck_kc;
                            PS_NOUNROLL_C for (int q = ws; q < we; ++q) { st[q - ws] = SWW(o_wt + (q)); su[q - ws] = SVW(o_wu + (q)); }
                        }
                        const int ws0 = ws, we0 = we;
                        we -= ws;
                        ws = 0;
                        uint32_t *rg = dst + ck_r + lane * CK_REGW;
                        if (has_stage) {
                            // the rows' band at this checkpoint (read by BAND restores and compares)
                            while (b_alo < b_hi && SW(o_Ai + (b_alo)) == A_DEAD) ++b_alo;
                            rg[21] = (uint32_t)b_alo;
                            rg[22] = (uint32_t)b_hi;
                        }
                        save_regs(rg);
                        *reinterpret_cast<long long *>(rg + 10) = (long long)segpk;
                        rg[9] = (uint32_t)max_win;     // widest window so far
                        rg[20] = (uint32_t)ecount;
                        segpk = 0;
                        ws = ws0;
                        we = we0;
                    } else {
                        ck_full = true;
                    }
                }
                if (REC && conv_c >= 0) break;
                __syncwarp();      // the checkpoint's reads before the commit's writes
            }
#if PS_SYNC_ARGMIN
            // Formal ordering for racecheck: other lanes' key reads of this
            // iteration before the commit's writes.  Off by default: the reads feed the argmin's
            // operands and the writes its result, and a converged warp's shared-memory accesses
            // complete in program order.
            __syncwarp();
#endif
            const int w = (int)((ml >> 24) & 63u);
            const int j = (int)((ml >> 2) & 0x3FFFFFu);
            const int k = (int)(ml & 3u);
            if (p.tcode && i == w) {
                p.tcode[(size_t)cand * p.tstride + ecount] = ml;
                p.tstart[(size_t)cand * p.tstride + ecount] = t;
            }
            if (REC && rank == RANK_COMPUTE && i == w) {
                p.cstep[i * L + pos] = (uint32_t)cc;
                if (k == KIND_F) p.fstep[i * m + j] = (uint32_t)cc;
            }
            ++ecount;
            if (rank == RANK_COMPUTE) ++cc;
            if (rank == RANK_COMPUTE) {
                if (i == w) {
                    const int end = t + proc_of(j, k);
                    rem -= end - t;
                    const bool newreq = derived && k == KIND_F && ((SB(o_offm + (j >> 5)) >> (j & 31)) & 1u);
                    win_insert(end, val_of(j, k));
                    sfree = end;
                    ++pos;
                    head = nxt;
                    nxt = fetch(pos + 1);
                    if (first_start == INT_MAX) first_start = t;
                    // End-time words keep their time only while a reader on another resource is to
                    // come; readers on the op's own stage are bounded by its free time, so there the
                    // time is dropped (canonical words).
                    if (k == KIND_F) {
                        // (every later write to row i, or row i's X, at microbatch j follows this F)
                        if (BAND || REC) b_hi = max(b_hi, j + 1);
                        SW(o_Ai + (j)) = ((uint32_t)end << 2) | 1u;
                        if (newreq) {
                            SB(o_poff + (j >> 5)) |= 1u << (j & 31);
                            ++n_poff;
                            if (wmask_on) pwm |= 1u << (j >> 5);
                        }
                        if (i > 0) {
                            // F(i, j) read A[i-1][j]; unless F(i-1, j)'s offload is still to come,
                            // only B(i-1, j) reads it now
                            const bool off_pending = ((SB(o_bits + (i - 1) * MW + (j >> 5)) >> (j & 31)) & 1u) &&
                                                     (SW(o_A + (P * m + (i - 1) * m + j)) & 3u) == 0u;
                            if (!off_pending) SW(o_A + ((i - 1) * m + j)) = 1u;
                        }
                    } else if (k == KIND_B) {
                        SW(o_Ai + (j)) = i == 0 ? 2u : (((uint32_t)end << 2) | 2u);   // B(i-1, j) reads it
                        SW(o_Xi + (j)) = 0u;                        // B(i, j) was its last reader
                        if (i + 1 < P) {
                            // B(i, j) read A[i+1][j]: W(i+1, j) remains (state 2) or nobody (state 3)
                            const uint32_t nb = SW(o_A + ((i + 1) * m + j));
                            SW(o_A + ((i + 1) * m + j)) = (nb & 3u) == 3u ? A_DEAD : 2u;
                        }
                    } else {
                        // W(i, j) is the last reader of A[i][j] unless B(i-1, j) is still to come
                        const bool up_done = i == 0 || (SW(o_A + ((i - 1) * m + j)) & 3u) >= 2u;
                        SW(o_Ai + (j)) = up_done ? A_DEAD : (SW(o_Ai + (j)) | 3u);
                    }
                    cdirty = true;
                    // reload keys read the ledger; a new request or explicit channel head may appear
                    tdirty = n_prel > 0 || newreq || !derived;
                } else if (k == KIND_F && i == w + 1) {
                    // F(w, j) only gates F(w+1, j)
                    cdirty = cdirty || (pos < L && head == (((uint32_t)j << 2) | KIND_F));
                } else if (k == KIND_B && i == w - 1) {
                    // B(w, j) only gates B(w-1, j)
                    cdirty = cdirty || (pos < L && head == (((uint32_t)j << 2) | KIND_B));
                }
            } else {
                const int end = t + p.toff;
                if (i == w) {
                    const V g = val_of(j, 3);
                    const uint32_t bit = 1u << (j & 31);
                    if (rank == RANK_OFFLOAD) {
                        // the reload's floor (this end) is bounded by the channel's free time: drop it;
                        // F(i, j)'s end keeps a reader only if F(i+1, j) is still to come
                        SW(o_Xi + (j)) = 1u;
                        if (i == P - 1 || (SW(o_A + ((i + 1) * m + j)) & 3u) != 0u) SW(o_Ai + (j)) = 1u;
                        win_insert(end, -g);
                        if (derived) {
                            const uint32_t rest = SB(o_poff + (j >> 5)) & ~bit;
                            SB(o_poff + (j >> 5)) = rest;
                            SB(o_prel + (j >> 5)) |= bit;
                            --n_poff; ++n_prel;
                            if (wmask_on) pwm = (pwm & ~(rest ? 0u : 1u << (j >> 5))) | (1u << (16 + (j >> 5)));
                        }
                    } else {
                        SW(o_Xi + (j)) = ((uint32_t)end << 2) | 2u;
                        win_insert(t, g);
                        --n_unrel;
                        if (derived) {
                            const uint32_t rest = SB(o_prel + (j >> 5)) & ~bit;
                            SB(o_prel + (j >> 5)) = rest;
                            --n_prel;
                            if (wmask_on && !rest) pwm &= ~(1u << (16 + (j >> 5)));
                        }
                    }
                    // the ledger changed: an F head re-fits; a B head may have been waiting on this reload
                    cdirty = cdirty || (pos < L && ((head & 3u) == KIND_F || head == (((uint32_t)j << 2) | KIND_B)));
                }
                const int wchan = __shfl_sync(0xffffffffu, chan_i, w);   // (warp-uniform branch)
                if (has_stage && chan_i == wchan) {
                    cfree = end;
                    tdirty = true;
                    if (!derived) {
                        if (REC && i == w) p.chstep[(size_t)chan_i * p.chan_stride + cpos] = (uint32_t)cc;
                        ++cpos;
                        chead = cnext;
                        cnext = fetch_chan(cpos + 1);
                    }
                }
            }
            __syncwarp();
        }

        // ================= finished or deadlocked =========================================
        if (REC && conv_c >= 0) {
            // The new base continues as the previous one, conv_delta later: its outcome is the
            // previous base's shifted, with this recording's peak prefix and early first starts.
            const int dl = conv_delta;
            const uint32_t fl = (uint32_t)p.base_info[1];
            const uint32_t *rgc = p.ck + (size_t)conv_c * p.ck_words + ck_r + lane * CK_REGW;
            const V sfx = (V)*reinterpret_cast<const long long *>(rgc + 18);   // previous base's S_c
            const int hi = has_stage ? (int)p.base_res[2 + P + i] + dl : 0;
            const int fs = !has_stage ? INT_MAX
                         : first_start != INT_MAX ? first_start : (int)p.base_res[2 + 2 * P + i] + dl;
            long long span = -1;
            if (fl == FLAG_FEASIBLE) {
                if (p.post) span = __reduce_max_sync(0xffffffffu, has_stage ? hi - fs : 0);
                else span = (long long)__reduce_max_sync(0xffffffffu, hi) - (long long)__reduce_min_sync(0xffffffffu, fs);
            }
            if (has_stage) {
                p.base_res[2 + i] = fl == FLAG_FEASIBLE ? (long long)(peak > sfx ? peak : sfx) * p.unit : -1;
                p.base_res[2 + P + i] = hi;
                p.base_res[2 + 2 * P + i] = fs;
                // suffix peaks of the checkpoints up to conv_c (later ones are unchanged)
                suffix_peaks(conv_c, (long long)sfx);
            }
            const int old_win = p.base_info[4], old_events = p.base_info[2];
            __syncwarp();
            if (lane == 0) {
                p.base_info[2] = old_events - eoff;    // its transfer events differ by eoff
                p.base_info[4] = max(max_win, old_win);
                p.base_info[5] = conv_c;
                p.base_info[6] = dl;
                p.base_info[7] = eoff;
                p.base_res[0] = span;
                double b = span > 0 ? 1.0 - (double)p.busy / ((double)P * (double)span)
                                    : __longlong_as_double(0x7ff8000000000000LL);
                p.base_res[1] = __double_as_longlong(b);
            }
            __syncwarp();
            continue;
        }
        if (conv_c >= 0) {
            // converged onto the base: its outcome, with this candidate's peak prefix
            const uint32_t fl = (uint32_t)p.base_info[1];
            if (p.peak && has_stage) {
                const V sfx = (V)*reinterpret_cast<const long long *>(p.ck + (size_t)conv_c * p.ck_words + ck_r + lane * CK_REGW + 18);
                p.peak[(size_t)cand * P + i] = fl == FLAG_FEASIBLE ? (long long)(peak > sfx ? peak : sfx) * p.unit : -1;
            }
            // the base's final free and first-start times, delta later (a stage that had started
            // keeps its own first start)
            long long span = -1;
            if (fl == FLAG_FEASIBLE) {
                const int hi = has_stage ? (int)p.base_res[2 + P + i] + conv_delta : 0;
                const int fs = !has_stage ? INT_MAX
                             : first_start != INT_MAX ? first_start : (int)p.base_res[2 + 2 * P + i] + conv_delta;
                if (p.post) span = __reduce_max_sync(0xffffffffu, has_stage ? hi - fs : 0);
                else span = (long long)__reduce_max_sync(0xffffffffu, hi) - (long long)__reduce_min_sync(0xffffffffu, fs);
            }
            if (lane == 0) {
                put_result(fl, span, (uint32_t)p.base_info[3], p.base_info[2] - eoff);
                if (MOVES && p.best_key && span >= 0) {
                    long long key = (span << 32) | (long long)(uint32_t)(p.first_index + cand);
                    if (key < *(volatile long long *)p.best_key) atomicMin(p.best_key, key);
                }
            }
            __syncwarp();
            continue;
        }
        if (pruned) {
            // cannot improve on the incumbent: no key, no outputs (search rounds request none)
            if (lane == 0 && p.events_total && ecount > ecount0)
                atomicAdd(p.events_total, (unsigned long long)(ecount - ecount0));
            __syncwarp();
            continue;
        }
        if (early_dl) {
            if (lane == 0) put_result(FLAG_DEADLOCK, -1LL, 0u, ecount);
            if (p.peak && has_stage) p.peak[(size_t)cand * P + i] = -1;
            __syncwarp();
            continue;
        }
        if (!REC && range_ovf) {
            if (lane == 0) put_result(FLAG_RANGE, -1LL, 0u, 0);
            if (p.peak && has_stage) p.peak[(size_t)cand * P + i] = -1;
            __syncwarp();
            continue;
        }
        const unsigned rem = __ballot_sync(0xffffffffu, has_stage && pos < L);
        if (REC) {
            const bool unusable = __any_sync(0xffffffffu, ovf || ck_full) || range_ovf;
            long long span = -1;
            if (!unusable && rem == 0u) {
                win_fold(INT_MAX);
                int hi = p.post ? (has_stage ? sfree - first_start : 0) : (has_stage ? sfree : 0);
                int lo = p.post ? 0 : (has_stage ? first_start : INT_MAX);
                span = (long long)__reduce_max_sync(0xffffffffu, hi) - (long long)__reduce_min_sync(0xffffffffu, lo);
            }
            if (has_stage) {
                p.base_res[2 + i] = rem == 0u ? (long long)peak * p.unit : -1;
                p.base_res[2 + P + i] = sfree;            // final free time and first start: a candidate
                p.base_res[2 + 2 * P + i] = first_start;  // converging with a time shift rebuilds its span
            }
            if (has_stage && rem != 0u) {
                // deadlocked base: what it never committed is NEVER (a resumed recording would
                // otherwise keep the previous base's steps there)
                for (int q = pos; q < L; ++q) p.cstep[i * L + q] = NEVER;
                if (!derived)      // (every lane of a channel writes the same entries)
                    for (int q = cpos; q < p.chan_stride; ++q) p.chstep[(size_t)chan_i * p.chan_stride + q] = NEVER;
                for (int j = 0; j < m; ++j)
                    if ((SW(o_Ai + (j)) & 3u) == 0u) p.fstep[i * m + j] = NEVER;
            }
            if (!unusable && has_stage) {
                // S_c = max usage folded after checkpoint c (a converging candidate's peak suffix)
                suffix_peaks(cc > 0 ? (cc - 1) / p.ck_interval : -1, (long long)segpk);
            }
            if (lane == 0) {
                p.base_info[5] = -1;                      // no shifted suffix to apply
                p.base_info[0] = unusable || cc == 0 ? -1 : (cc - 1) / p.ck_interval + 1;
                p.base_info[4] = max_win;
                p.base_info[1] = (int)(rem == 0u ? FLAG_FEASIBLE : range_ovf ? FLAG_RANGE : FLAG_DEADLOCK);
                p.base_info[2] = ecount;
                p.base_info[3] = (int)rem;
                p.base_res[0] = span;
                double b = span > 0 ? 1.0 - (double)p.busy / ((double)P * (double)span)
                                    : __longlong_as_double(0x7ff8000000000000LL);
                p.base_res[1] = __double_as_longlong(b);
            }
        } else if (__any_sync(0xffffffffu, ovf)) {
            if (lane == 0 && p.ovf_list) {
                int at = atomicAdd(p.ovf_count, 1);
                p.ovf_list[at] = (int32_t)cand;
            }
        } else if (rem == 0u) {
            win_fold(INT_MAX);
            int hi, lo;
            if (p.post) {
                hi = has_stage ? sfree - first_start : 0;
                lo = 0;
            } else {
                hi = has_stage ? sfree : 0;
                lo = has_stage ? first_start : INT_MAX;
            }
            hi = __reduce_max_sync(0xffffffffu, hi);
            lo = __reduce_min_sync(0xffffffffu, lo);
            const long long span = (long long)hi - (long long)lo;
            if (p.peak && has_stage) p.peak[(size_t)cand * P + i] = (long long)peak * p.unit;
            if (lane == 0) {
                put_result(FLAG_FEASIBLE, span, 0u, 0);
                if (MOVES && p.best_key) {
                    long long key = (span << 32) | (long long)(uint32_t)(p.first_index + cand);
                    if (key < *(volatile long long *)p.best_key) atomicMin(p.best_key, key);
                }
            }
        } else {
            if (lane == 0) put_result(FLAG_DEADLOCK, -1LL, rem, ecount);
            if (p.peak && has_stage) p.peak[(size_t)cand * P + i] = -1;
        }
        __syncwarp();
    }
#undef SW
#undef SV
#undef SB
#undef SWW
#undef SVW
}

}  // namespace ps
