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

constexpr uint32_t FLAG_FEASIBLE = 1u, FLAG_DEADLOCK = 2u, FLAG_MALFORMED = 4u, FLAG_OVERFLOW = 8u;
constexpr int TAU_NONE = INT_MAX;   // usage never drops far enough: earliest_fit returns None
constexpr int TAU_ANY = INT_MIN;    // fits at any query time at or above the fold line
constexpr uint32_t NO_CHAN = 0xFFFFFFFFu;

struct EvalParams {
    // instance (device tables)
    int P, m, G, L, MW, stride;
    int comm, toff, post, uniform, any_off;
    int64_t busy, unit;
    const int32_t *proc;     // [rows][3]
    const void *vals;        // V [rows][4] = dF, dB, dW, gamma (in memory units)
    const void *limit;       // V [P]
    const int32_t *chan;     // [P]
    // materialised candidates
    int64_t N;
    const uint16_t *orders;
    const uint32_t *masks;
    const uint32_t *chorders;
    int chan_stride;
    // move-encoded candidates (search)
    const uint16_t *inc_orders;
    const uint32_t *inc_mask;
    uint64_t seed, round;
    int64_t first_index;
    uint32_t shift_permille, max_shift;
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
    const int32_t *work_list;
    const int32_t *work_count;
    // per-candidate state
    int K;                   // ledger window capacity (power of two)
    int cand_words;          // 32-bit words of one candidate's state
    int inc_words;           // 32-bit words of the block-shared incumbent (move mode)
    uint32_t *gstate;        // GSTATE scratch
};

template <typename V>
__device__ __forceinline__ V ldv(const void *base, int idx) {
    return __ldg(reinterpret_cast<const V *>(base) + idx);
}

__device__ __forceinline__ bool key_less(uint32_t ah, uint32_t al, uint32_t bh, uint32_t bl) {
    return ah < bh || (ah == bh && al < bl);
}

template <typename V, bool MOVES, bool GSTATE>
__global__ void __launch_bounds__(128) eval_kernel(const EvalParams p) {
    extern __shared__ __align__(16) uint32_t smem[];
    constexpr int VW = sizeof(V) / 4;
    const int lane = threadIdx.x & 31;
    const int warp = threadIdx.x >> 5;
    const int nwarps = blockDim.x >> 5;
    const int P = p.P, m = p.m, L = p.L, MW = p.MW, K = p.K, KM = p.K - 1;
    const int i = lane;                               // the stage this lane owns
    const bool has_stage = i < P;
    const int is = has_stage ? i : 0;
    const bool derived = p.chorders == nullptr;

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
    uint32_t *cb = GSTATE ? p.gstate + (size_t)slot * p.cand_words : smem + p.inc_words + (size_t)warp * p.cand_words;
    V *wd = reinterpret_cast<V *>(cb) + (size_t)is * K;                 // own ledger window: deltas
    uint32_t *wt = cb + (size_t)P * K * VW + (size_t)is * K;              // own ledger window: times
    uint32_t *A = cb + (size_t)P * K * (VW + 1);         // [P][m] F end, then B end   (time<<2 | state)
    uint32_t *X = A + (size_t)P * m;                      // [P][m] offload end, then reload end
    uint32_t *offm = X + (size_t)P * m;                   // [P][MW] offloaded bits
    uint32_t *poff = offm + (size_t)P * MW;               // [P][MW] pending offload requests
    uint32_t *prel = poff + (size_t)P * MW;               // [P][MW] pending reload requests
    uint32_t *A_i = A + (size_t)is * m;
    uint32_t *X_i = X + (size_t)is * m;
    uint32_t *offm_i = offm + is * MW;
    uint32_t *poff_i = poff + is * MW;
    uint32_t *prel_i = prel + is * MW;
    const int nz = 2 * P * m + 3 * P * MW;               // words zeroed per candidate

    const int chan_i = has_stage ? __ldg(&p.chan[i]) : -1;
    const V limit_i = has_stage ? ldv<V>(p.limit, i) : V(0);
    const int rowbase = p.uniform ? is : is * m;
    // per-stage constants of microbatch-symmetric instances live in registers
    int t0 = 0, t1 = 0, t2 = 0;
    V v0 = 0, v1 = 0, v2 = 0, v3 = 0;
    if (p.uniform) {
        t0 = __ldg(&p.proc[rowbase * 3 + 0]);
        t1 = __ldg(&p.proc[rowbase * 3 + 1]);
        t2 = __ldg(&p.proc[rowbase * 3 + 2]);
        v0 = ldv<V>(p.vals, rowbase * 4 + 0);
        v1 = ldv<V>(p.vals, rowbase * 4 + 1);
        v2 = ldv<V>(p.vals, rowbase * 4 + 2);
        v3 = ldv<V>(p.vals, rowbase * 4 + 3);
    }
    auto proc_of = [&](int j, int k) -> int {
        if (p.uniform) return k == 0 ? t0 : (k == 1 ? t1 : t2);
        return __ldg(&p.proc[(rowbase + j) * 3 + k]);
    };
    auto val_of = [&](int j, int k) -> V {
        if (p.uniform) return k == 0 ? v0 : (k == 1 ? v1 : (k == 2 ? v2 : v3));
        return ldv<V>(p.vals, (rowbase + j) * 4 + k);
    };

    // ---- per-lane registers ----------------------------------------------------------------
    long long cand = 0;
    Move mv;
    mv.type = MOVE_NOOP; mv.stage = 0; mv.a = mv.b = 0; mv.mb = 0;
    int pos = 0, sfree = 0, cfree = 0;
    uint32_t ckh = KEY_NONE, ckl = KEY_NONE;   // cached compute-head key
    uint32_t tkh = KEY_NONE, tkl = KEY_NONE;   // cached best transfer key of this stage
    bool cdirty = false, tdirty = false, ovf = false;
    V base = 0, top = 0, peak = 0;
    int wh = 0, wn = 0;
    int n_poff = 0, n_prel = 0, n_unrel = 0;   // pending offloads / reloads / offloaded not yet reloaded
    V rF = V(-1), rG = V(-1);                  // earliest_fit cache, valid until the ledger changes
    int tauF = 0, tauG = 0;
    int first_start = INT_MAX, first_f = INT_MAX, last_w = 0;
    int ecount = 0;
    uint32_t head = 0, nxt = 0;
    int cpos = 0;
    uint32_t chead = NO_CHAN, cnext = NO_CHAN;

    auto fetch = [&](int q) -> uint32_t {
        if (q >= L || !has_stage) return 0u;
        if (MOVES) {
            int src = (mv.type == MOVE_SHIFT && i == mv.stage) ? shifted_position(q, mv.a, mv.b) : q;
            return inc_s[i * p.stride + src];
        }
        return __ldg(&p.orders[((size_t)cand * P + i) * p.stride + q]);
    };
    auto fetch_chan = [&](int q) -> uint32_t {
        if (derived || !has_stage || q >= p.chan_stride) return NO_CHAN;
        return __ldg(&p.chorders[((size_t)cand * p.G + chan_i) * p.chan_stride + q]);
    };

    // Ledger window: ring of K (time, delta) points sorted by time, all >= the fold line.
    auto win_fold = [&](int line) {
        while (wn > 0 && (int)wt[wh] < line) {
            int t = (int)wt[wh];
            do {
                base += wd[wh];
                wh = (wh + 1) & KM;
                --wn;
            } while (wn > 0 && (int)wt[wh] == t);
            peak = base > peak ? base : peak;
        }
    };
    // Called before sfree / cfree / n_unrel reflect the event being committed: the fold line is
    // below sfree, and below the channel's free time while this stage still has a transfer to come,
    // so no future query or insertion (this one included) lands under it.
    auto win_insert = [&](int t, V d) {
        win_fold(n_unrel > 0 ? min(sfree, cfree) : sfree);
        top += d;
        rF = rG = V(-1);                               // the ledger changed: drop cached answers
        if (wn == K) { ovf = true; return; }
        int k = wn;
        while (k > 0) {
            int src = (wh + k - 1) & KM;
            if ((int)wt[src] <= t) break;
            int dst = (wh + k) & KM;
            wt[dst] = wt[src];
            wd[dst] = wd[src];
            --k;
        }
        int dst = (wh + k) & KM;
        wt[dst] = (uint32_t)t;
        wd[dst] = d;
        ++wn;
    };
    // earliest_fit core: first breakpoint after the last one whose usage exceeds R.
    auto win_tau = [&](V R) -> int {
        if (R < 0) return TAU_NONE;
        V u = top;
        if (u > R) return TAU_NONE;
        int k = wn - 1;
        while (k >= 0) {
            int t = (int)wt[(wh + k) & KM];
            do {
                u -= wd[(wh + k) & KM];
                --k;
            } while (k >= 0 && (int)wt[(wh + k) & KM] == t);
            if (u > R) return t;
        }
        return TAU_ANY;
    };
    auto tau_F = [&](V R) -> int {
        if (R != rF) { tauF = win_tau(R); rF = R; }
        return tauF;
    };
    auto tau_G = [&](V R) -> int {
        if (R != rG) { tauG = win_tau(R); rG = R; }
        return tauG;
    };

    auto compute_key = [&]() {
        ckh = ckl = KEY_NONE;
        if (pos >= L) return;
        const int j = head >> 2, k = head & 3u;
        int fl;
        if (k == KIND_F) {
            fl = 0;
            if (i > 0) {
                uint32_t a = A[(i - 1) * m + j];
                if (!(a & 3u)) return;
                fl = (int)(a >> 2) + p.comm;
            }
        } else if (k == KIND_B) {
            uint32_t a = A_i[j];
            if ((a & 3u) != 1u) return;
            fl = (int)(a >> 2);
            if (i < P - 1) {
                uint32_t b = A[(i + 1) * m + j];
                if ((b & 3u) != 2u) return;
                fl = max(fl, (int)(b >> 2) + p.comm);
            }
            if ((offm_i[j >> 5] >> (j & 31)) & 1u) {
                uint32_t x = X_i[j];
                if ((x & 3u) != 2u) return;
                fl = max(fl, (int)(x >> 2));
            }
        } else {
            uint32_t a = A_i[j];
            if ((a & 3u) != 2u) return;
            fl = (int)(a >> 2);
        }
        int lo = max(fl, sfree);
        if (k == KIND_F) {
            int tau = tau_F(limit_i - val_of(j, 0));
            if (tau == TAU_NONE) return;
            if (tau != TAU_ANY) lo = max(lo, tau - proc_of(j, 0));
        }
        ckh = (uint32_t)lo;
        ckl = ((uint32_t)i << 24) | ((uint32_t)j << 2) | (uint32_t)k;
    };

    auto transfer_key = [&]() {
        uint32_t bh = KEY_NONE, bl = KEY_NONE;
        const int C = cfree;
        const uint32_t sb = (uint32_t)i << 24;
        if (derived) {
            if (n_poff)
                for (int w = 0; w < MW; ++w)
                    for (uint32_t bits = poff_i[w]; bits; bits &= bits - 1) {
                        int j = w * 32 + __ffs(bits) - 1;
                        uint32_t h = (uint32_t)max((int)(A_i[j] >> 2), C), l = (2u << 30) | sb | ((uint32_t)j << 2);
                        if (key_less(h, l, bh, bl)) { bh = h; bl = l; }
                    }
            if (n_prel)
                for (int w = 0; w < MW; ++w)
                    for (uint32_t bits = prel_i[w]; bits; bits &= bits - 1) {
                        int j = w * 32 + __ffs(bits) - 1;
                        int tau = tau_G(limit_i - val_of(j, 3));
                        if (tau == TAU_NONE) continue;
                        uint32_t h = (uint32_t)max(max((int)(X_i[j] >> 2), C), tau);
                        uint32_t l = (1u << 30) | sb | ((uint32_t)j << 2);
                        if (key_less(h, l, bh, bl)) { bh = h; bl = l; }
                    }
        } else if (chead != NO_CHAN && (int)((chead >> 16) & 0x7FFFu) == i) {
            int j = chead & 0xFFFFu;
            if (!(chead >> 31)) {
                uint32_t a = A_i[j];
                if (a & 3u) { bh = (uint32_t)max((int)(a >> 2), C); bl = (2u << 30) | sb | ((uint32_t)j << 2); }
            } else {
                uint32_t x = X_i[j];
                if ((x & 3u) == 1u) {
                    int tau = tau_G(limit_i - val_of(j, 3));
                    if (tau != TAU_NONE) {
                        bh = (uint32_t)max(max((int)(x >> 2), C), tau);
                        bl = (1u << 30) | sb | ((uint32_t)j << 2);
                    }
                }
            }
        }
        tkh = bh;
        tkl = bl;
    };

    // Lane 0 publishes a candidate's outcome (search rounds may pass no arrays).
    auto put_result = [&](uint32_t flag, long long span, uint32_t blocked_mask) {
        if (p.events_total && ecount) atomicAdd(p.events_total, (unsigned long long)ecount);
        if (p.flags) p.flags[cand] = flag;
        if (p.makespan) p.makespan[cand] = span;
        if (p.bubble)
            p.bubble[cand] = span > 0 ? 1.0 - (double)p.busy / ((double)P * (double)span)
                                      : __longlong_as_double(0x7ff8000000000000LL);
        if (p.blocked) p.blocked[cand] = blocked_mask;
    };

    const long long n_items = p.work_list ? (long long)*p.work_count : p.N;
    for (long long item = slot; item < n_items; item += nslots) {
        cand = p.work_list ? (long long)p.work_list[item] : item;
        // ================= initialise ======================================================
        for (int k = lane; k < nz; k += 32) A[k] = 0u;
        if (MOVES) {
            uint64_t gidx = (uint64_t)(p.first_index + cand);
            mv = decode_move(p.seed, p.round, gidx, P, m, p.shift_permille, p.max_shift, p.any_off != 0,
                             [&](int s, int j) { return ldv<V>(p.vals, (p.uniform ? s : s * m + j) * 4 + 3) > V(0); });
        }
        __syncwarp();
        bool bad = false;
        n_unrel = 0;
        if (has_stage) {
            const int mwords = (P * m + 31) / 32;
            for (int w = 0; w < MW; ++w) {
                // bits [i*m + 32w, i*m + 32w + 32) of the packed candidate mask
                const int gb = i * m + w * 32, q = gb >> 5, sh = gb & 31;
                auto word = [&](int qq) -> uint32_t {
                    if (qq >= mwords) return 0u;
                    return MOVES ? incmask_s[qq] : __ldg(&p.masks[(size_t)cand * mwords + qq]);
                };
                uint32_t bits = word(q) >> sh;
                if (sh) bits |= word(q + 1) << (32 - sh);
                const int nb = m - w * 32;
                if (nb < 32) bits &= (1u << nb) - 1u;
                if (MOVES && mv.type == MOVE_TOGGLE && mv.stage == i && (mv.mb >> 5) == w) bits ^= 1u << (mv.mb & 31);
                offm_i[w] = bits;
                n_unrel += __popc(bits);
                // an offload bit on a non-offloadable op is malformed (KeyError in the reference)
                for (uint32_t t = bits; t; t &= t - 1)
                    if (!(val_of(w * 32 + __ffs(t) - 1, 3) > 0)) bad = true;
            }
            if (!MOVES) {
                // the stage order must be a permutation of the stage's 3m ops
                for (int q = 0; q < L; ++q) {
                    uint32_t op = __ldg(&p.orders[((size_t)cand * P + i) * p.stride + q]);
                    uint32_t j = op >> 2, k = op & 3u;
                    if (j >= (uint32_t)m || k > 2u || (A_i[j] >> k) & 1u) { bad = true; break; }
                    A_i[j] |= 1u << k;
                }
                if (!bad)
                    for (int j = 0; j < m; ++j)
                        if (A_i[j] != 7u) { bad = true; break; }
                for (int j = 0; j < m; ++j) A_i[j] = 0u;
            }
        }
        if (__any_sync(0xffffffffu, bad)) {
            if (lane == 0) put_result(FLAG_MALFORMED, -1LL, 0u);
            __syncwarp();
            continue;
        }
        pos = 0; sfree = 0; cfree = 0; ovf = false;
        base = top = peak = 0; wh = wn = 0;
        n_poff = n_prel = 0;
        rF = rG = V(-1);
        first_start = INT_MAX; first_f = INT_MAX; last_w = 0; ecount = 0;
        head = fetch(0); nxt = fetch(1);
        cpos = 0; chead = fetch_chan(0); cnext = fetch_chan(1);
        cdirty = tdirty = has_stage;
        ckh = ckl = tkh = tkl = KEY_NONE;
        __syncwarp();

        // ================= simulate: one committed event per iteration ===================
        for (;;) {
            if (cdirty) { compute_key(); cdirty = false; }
            if (tdirty) { transfer_key(); tdirty = false; }
            uint32_t kh = ckh, kl = ckl;
            if (key_less(tkh, tkl, kh, kl)) { kh = tkh; kl = tkl; }
            const uint32_t mh = __reduce_min_sync(0xffffffffu, kh);
            const uint32_t ml = __reduce_min_sync(0xffffffffu, kh == mh ? kl : 0xFFFFFFFFu);
            if (mh == KEY_NONE) break;

            const int t = (int)mh;
            const int rank = (int)(ml >> 30);
            const int w = (int)((ml >> 24) & 63u);
            const int j = (int)((ml >> 2) & 0x3FFFFFu);
            const int k = (int)(ml & 3u);
            if (p.tcode && i == w) {
                p.tcode[(size_t)cand * p.tstride + ecount] = ml;
                p.tstart[(size_t)cand * p.tstride + ecount] = t;
            }
            ++ecount;
            if (rank == RANK_COMPUTE) {
                if (i == w) {
                    const int end = t + proc_of(j, k);
                    const bool newreq = derived && k == KIND_F && ((offm_i[j >> 5] >> (j & 31)) & 1u);
                    win_insert(end, val_of(j, k));
                    sfree = end;
                    ++pos;
                    head = nxt;
                    nxt = fetch(pos + 1);
                    if (first_start == INT_MAX) first_start = t;
                    if (k == KIND_F) {
                        A_i[j] = ((uint32_t)end << 2) | 1u;
                        if (first_f == INT_MAX) first_f = t;
                        if (newreq) { poff_i[j >> 5] |= 1u << (j & 31); ++n_poff; }
                    } else if (k == KIND_B) {
                        A_i[j] = ((uint32_t)end << 2) | 2u;
                    } else {
                        last_w = end;
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
                        X_i[j] = ((uint32_t)end << 2) | 1u;
                        win_insert(end, -g);
                        if (derived) { poff_i[j >> 5] &= ~bit; prel_i[j >> 5] |= bit; --n_poff; ++n_prel; }
                    } else {
                        X_i[j] = ((uint32_t)end << 2) | 2u;
                        win_insert(t, g);
                        --n_unrel;
                        if (derived) { prel_i[j >> 5] &= ~bit; --n_prel; }
                    }
                    // the ledger changed: an F head re-fits; a B head may have been waiting on this reload
                    cdirty = cdirty || (pos < L && ((head & 3u) == KIND_F || head == (((uint32_t)j << 2) | KIND_B)));
                }
                if (has_stage && chan_i == __ldg(&p.chan[w])) {
                    cfree = end;
                    tdirty = true;
                    if (!derived) {
                        ++cpos;
                        chead = cnext;
                        cnext = fetch_chan(cpos + 1);
                    }
                }
            }
            __syncwarp();
        }

        // ================= finished or deadlocked =========================================
        const unsigned rem = __ballot_sync(0xffffffffu, has_stage && pos < L);
        if (__any_sync(0xffffffffu, ovf)) {
            if (lane == 0 && p.ovf_list) {
                int at = atomicAdd(p.ovf_count, 1);
                p.ovf_list[at] = (int32_t)cand;
            }
        } else if (rem == 0u) {
            win_fold(INT_MAX);
            int hi, lo;
            if (p.post) {
                hi = has_stage ? last_w - first_f : 0;
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
                put_result(FLAG_FEASIBLE, span, 0u);
                if (MOVES && p.best_key) {
                    long long key = (span << 32) | (long long)(uint32_t)(p.first_index + cand);
                    if (key < *(volatile long long *)p.best_key) atomicMin(p.best_key, key);
                }
            }
        } else {
            if (lane == 0) put_result(FLAG_DEADLOCK, -1LL, rem);
            if (p.peak && has_stage) p.peak[(size_t)cand * P + i] = -1;
        }
        __syncwarp();
    }
}

}  // namespace ps
