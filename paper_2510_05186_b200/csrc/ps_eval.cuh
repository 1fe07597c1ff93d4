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
//   * one lane per stage, SEG = next pow2 >= P lanes per candidate, 32/SEG candidates per warp, each
//     segment streaming its own sequence of candidates (no tail waiting on the slowest neighbour);
//   * each lane caches its stage's best key (compute head or transfer option of that stage) and
//     recomputes it only when the committed event can have changed it; the global argmin is a
//     segment butterfly over 64-bit keys (start:32 | rank:2 stage:6 microbatch:22 kind:2);
//   * the stage ledger is folded below a monotone frontier (no future query or insertion can land
//     there), so only a short window of future points stays live in shared memory; earliest_fit
//     becomes a backward scan for the last breakpoint whose usage exceeds limit - delta
//     (SURVEY.md A.3), exact;
//   * per-(stage, microbatch) end times are packed as (time << 2 | state) words in shared memory;
//   * a candidate whose window overflows is re-run by the GSTATE variant (state in global memory,
//     window = 5m, never overflows) from a device-side worklist — no host round trip, no CPU path.
#pragma once
#include <stdint.h>
#include <climits>
#include "ps_common.cuh"

namespace ps {

constexpr uint32_t FLAG_FEASIBLE = 1u, FLAG_DEADLOCK = 2u, FLAG_MALFORMED = 4u, FLAG_OVERFLOW = 8u;
constexpr int TAU_NONE = INT_MAX;   // usage never drops far enough: earliest_fit returns None
constexpr int TAU_ANY = INT_MIN;    // fits at any query time at or above the fold line

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

template <int SEG, typename V, bool MOVES, bool GSTATE>
__global__ void __launch_bounds__(128) eval_kernel(const EvalParams p) {
    extern __shared__ __align__(16) uint32_t smem[];
    constexpr int SEGS = 32 / SEG;
    constexpr int VW = sizeof(V) / 4;
    const int lane = threadIdx.x & 31;
    const int warp = threadIdx.x >> 5;
    const int nwarps = blockDim.x >> 5;
    const int seg = lane / SEG;
    const int i = lane % SEG;                       // the stage this lane owns
    const unsigned segmask = SEG == 32 ? 0xffffffffu : (((1u << SEG) - 1u) << (seg * SEG));
    const int P = p.P, m = p.m, L = p.L, MW = p.MW, K = p.K, KM = p.K - 1;
    const bool has_stage = i < P;
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

    // ---- this segment's state slot --------------------------------------------------------
    const long long slot = ((long long)blockIdx.x * nwarps + warp) * SEGS + seg;
    const long long nslots = (long long)gridDim.x * nwarps * SEGS;
    uint32_t *cb = GSTATE ? p.gstate + (size_t)slot * p.cand_words
                          : smem + p.inc_words + (size_t)(warp * SEGS + seg) * p.cand_words;
    V *wd = reinterpret_cast<V *>(cb) + (size_t)(has_stage ? i : 0) * K;   // own window deltas
    uint32_t *wt = cb + (size_t)P * K * VW + (size_t)(has_stage ? i : 0) * K;
    uint32_t *A = cb + (size_t)P * K * (VW + 1);         // [P][m] F end, then B end
    uint32_t *X = A + (size_t)P * m;                      // [P][m] offload end, then reload end
    uint32_t *offm = X + (size_t)P * m;                   // [P][MW] offloaded bits
    uint32_t *poff = offm + (size_t)P * MW;               // [P][MW] pending offload requests
    uint32_t *prel = poff + (size_t)P * MW;               // [P][MW] pending reload requests
    uint32_t *A_i = A + (size_t)(has_stage ? i : 0) * m;
    uint32_t *X_i = X + (size_t)(has_stage ? i : 0) * m;
    uint32_t *offm_i = offm + (has_stage ? i : 0) * MW;
    uint32_t *poff_i = poff + (has_stage ? i : 0) * MW;
    uint32_t *prel_i = prel + (has_stage ? i : 0) * MW;

    const int chan_i = has_stage ? __ldg(&p.chan[i]) : -1;
    const V limit_i = has_stage ? ldv<V>(p.limit, i) : V(0);
    const int rowbase = p.uniform ? i : i * m;

    // ---- per-lane registers ----------------------------------------------------------------
    long long n_items = p.work_list ? (long long)*p.work_count : p.N;
    long long item = slot - nslots;
    long long cand = 0;
    bool alive = false;
    int pos = 0, sfree = 0, cfree = 0;
    uint32_t khi = KEY_NONE, klo = KEY_NONE;
    bool dirty = false, ovf = false;
    V base = 0, top = 0, peak = 0;
    int wh = 0, wn = 0;
    int first_start = INT_MAX, first_f = INT_MAX, last_w = 0;
    int ecount = 0;
    uint32_t head = 0, nxt = 0;      // current / next op code of this stage
    int cpos = 0;                    // explicit channel mode: position in this lane's channel order
    uint32_t chead = 0xFFFFFFFFu, cnext = 0xFFFFFFFFu;
    Move mv;
    mv.type = MOVE_NOOP; mv.stage = 0; mv.a = mv.b = 0; mv.mb = 0;

    auto fetch = [&](int q) -> uint32_t {
        if (q >= L || !has_stage) return 0u;
        if (MOVES) {
            int src = (mv.type == MOVE_SHIFT && i == mv.stage) ? shifted_position(q, mv.a, mv.b) : q;
            return inc_s[i * p.stride + src];
        }
        return __ldg(&p.orders[((size_t)cand * P + i) * p.stride + q]);
    };
    auto fetch_chan = [&](int q) -> uint32_t {
        if (derived || !has_stage || q >= p.chan_stride) return 0xFFFFFFFFu;
        return __ldg(&p.chorders[((size_t)cand * p.G + chan_i) * p.chan_stride + q]);
    };
    auto proc_of = [&](int j, int k) -> int { return __ldg(&p.proc[(p.uniform ? rowbase : rowbase + j) * 3 + k]); };
    auto val_of = [&](int j, int k) -> V { return ldv<V>(p.vals, (p.uniform ? rowbase : rowbase + j) * 4 + k); };

    // Lane 0 of a segment publishes a candidate's outcome (search rounds may pass no arrays).
    auto put_result = [&](uint32_t flag, long long span, uint32_t blocked_mask) {
        if (p.flags) p.flags[cand] = flag;
        if (p.makespan) p.makespan[cand] = span;
        if (p.bubble)
            p.bubble[cand] = span > 0 ? 1.0 - (double)p.busy / ((double)P * (double)span)
                                      : __longlong_as_double(0x7ff8000000000000LL);
        if (p.blocked) p.blocked[cand] = blocked_mask;
    };

    // Ledger window: ring of K (time, delta) points sorted by time, all >= the fold line.
    auto win_insert = [&](int t, V d) {
        top += d;
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
    auto win_fold = [&](int tmin) {
        while (wn > 0 && (int)wt[wh] < tmin) {
            int t = (int)wt[wh];
            do {
                base += wd[wh];
                wh = (wh + 1) & KM;
                --wn;
            } while (wn > 0 && (int)wt[wh] == t);
            peak = base > peak ? base : peak;
        }
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

    for (;;) {
        // ================= fetch / initialise a candidate for an idle segment =================
        if (!alive) {
            item += nslots;
            if (item < n_items) {
                cand = p.work_list ? (long long)p.work_list[item] : item;
                alive = true;
                // zero the candidate's A, X and bit sets (lanes of the segment cooperate)
                int nz = 2 * P * m + 3 * P * MW;
                for (int k = i; k < nz; k += SEG) A[k] = 0u;
                if (MOVES) {
                    uint64_t gidx = (uint64_t)(p.first_index + cand);
                    mv = decode_move(p.seed, p.round, gidx, P, m, p.shift_permille, p.max_shift,
                                     p.any_off != 0, [&](int s, int j) {
                                         return ldv<V>(p.vals, (p.uniform ? s : s * m + j) * 4 + 3) > V(0);
                                     });
                }
                __syncwarp(segmask);
                bool bad = false;
                if (has_stage) {
                    // offloaded bits of this stage, re-based to [MW] words
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
                        if (MOVES && mv.type == MOVE_TOGGLE && mv.stage == i && (mv.mb >> 5) == w)
                            bits ^= 1u << (mv.mb & 31);
                        offm_i[w] = bits;
                        // an offload bit on a non-offloadable op is malformed (KeyError in the reference)
                        for (uint32_t t = bits; t; t &= t - 1) {
                            int j = w * 32 + __ffs(t) - 1;
                            if (!(val_of(j, 3) > 0)) bad = true;
                        }
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
                pos = 0; sfree = 0; cfree = 0; dirty = true; ovf = false;
                base = top = peak = 0; wh = wn = 0;
                first_start = INT_MAX; first_f = INT_MAX; last_w = 0; ecount = 0;
                khi = klo = KEY_NONE;
                head = fetch(0); nxt = fetch(1);
                cpos = 0; chead = fetch_chan(0); cnext = fetch_chan(1);
                if (__any_sync(segmask, bad)) {
                    if (i == 0) put_result(FLAG_MALFORMED, -1LL, 0u);
                    alive = false;
                }
                __syncwarp(segmask);
            }
        }
        if (!__any_sync(0xffffffffu, alive || item < n_items)) break;

        // ================= recompute this stage's best key if it may have changed =============
        if (alive && has_stage && dirty) {
            dirty = false;
            uint32_t bhi = KEY_NONE, blo = KEY_NONE;
            auto consider = [&](int t, uint32_t lo) {
                uint32_t h = (uint32_t)t;
                if (h < bhi || (h == bhi && lo < blo)) { bhi = h; blo = lo; }
            };
            const int C = cfree;
            int tmin = sfree;
            const uint32_t stage_bits = (uint32_t)i << 24;
            if (derived) {
                for (int w = 0; w < MW; ++w) {
                    for (uint32_t bits = poff_i[w]; bits; bits &= bits - 1) {
                        int j = w * 32 + __ffs(bits) - 1;
                        int lo = max((int)(A_i[j] >> 2), C);
                        tmin = min(tmin, lo);
                        consider(lo, (2u << 30) | stage_bits | ((uint32_t)j << 2));
                    }
                    for (uint32_t bits = prel_i[w]; bits; bits &= bits - 1) {
                        int j = w * 32 + __ffs(bits) - 1;
                        tmin = min(tmin, max((int)(X_i[j] >> 2), C));
                    }
                }
            } else {
                if (chead != 0xFFFFFFFFu && (int)((chead >> 16) & 0x7FFFu) == i) {
                    int j = chead & 0xFFFFu;
                    if (!(chead >> 31)) {
                        uint32_t a = A_i[j];
                        if (a & 3u) {
                            int lo = max((int)(a >> 2), C);
                            consider(lo, (2u << 30) | stage_bits | ((uint32_t)j << 2));
                        }
                    }
                }
                // every future transfer of this stage starts at or after these bounds
                for (int w = 0; w < MW; ++w)
                    for (uint32_t bits = offm_i[w]; bits; bits &= bits - 1) {
                        int j = w * 32 + __ffs(bits) - 1;
                        uint32_t x = X_i[j];
                        if ((x & 3u) == 2u) continue;
                        if ((x & 3u) == 1u) tmin = min(tmin, max((int)(x >> 2), C));
                        else if (A_i[j] & 3u) tmin = min(tmin, max((int)(A_i[j] >> 2), C));
                    }
            }
            win_fold(tmin);
            if (derived) {
                V lastg = V(-1);
                int tau = TAU_NONE;
                for (int w = 0; w < MW; ++w)
                    for (uint32_t bits = prel_i[w]; bits; bits &= bits - 1) {
                        int j = w * 32 + __ffs(bits) - 1;
                        V g = val_of(j, 3);
                        if (g != lastg) { tau = win_tau(limit_i - g); lastg = g; }
                        if (tau == TAU_NONE) continue;
                        int lo = max(max((int)(X_i[j] >> 2), C), tau);
                        consider(lo, (1u << 30) | stage_bits | ((uint32_t)j << 2));
                    }
            } else if (chead != 0xFFFFFFFFu && (chead >> 31) && (int)((chead >> 16) & 0x7FFFu) == i) {
                int j = chead & 0xFFFFu;
                uint32_t x = X_i[j];
                if ((x & 3u) == 1u) {
                    int tau = win_tau(limit_i - val_of(j, 3));
                    if (tau != TAU_NONE)
                        consider(max(max((int)(x >> 2), C), tau), (1u << 30) | stage_bits | ((uint32_t)j << 2));
                }
            }
            if (pos < L) {
                const int j = head >> 2, k = head & 3u;
                bool ok = true;
                int fl = 0;
                if (k == KIND_F) {
                    if (i > 0) {
                        uint32_t a = A[(i - 1) * m + j];
                        ok = (a & 3u) != 0u;
                        fl = (int)(a >> 2) + p.comm;
                    }
                } else if (k == KIND_B) {
                    uint32_t a = A_i[j];
                    ok = (a & 3u) == 1u;
                    fl = (int)(a >> 2);
                    if (i < P - 1) {
                        uint32_t b = A[(i + 1) * m + j];
                        ok = ok && (b & 3u) == 2u;
                        fl = max(fl, (int)(b >> 2) + p.comm);
                    }
                    if ((offm_i[j >> 5] >> (j & 31)) & 1u) {
                        uint32_t x = X_i[j];
                        ok = ok && (x & 3u) == 2u;
                        fl = max(fl, (int)(x >> 2));
                    }
                } else {
                    uint32_t a = A_i[j];
                    ok = (a & 3u) == 2u;
                    fl = (int)(a >> 2);
                }
                if (ok) {
                    int lo = max(fl, sfree);
                    if (k == KIND_F) {
                        int tau = win_tau(limit_i - val_of(j, 0));
                        if (tau == TAU_NONE) ok = false;
                        else if (tau != TAU_ANY) lo = max(lo, tau - proc_of(j, 0));
                    }
                    if (ok) consider(lo, stage_bits | ((uint32_t)j << 2) | (uint32_t)k);
                }
            }
            khi = bhi;
            klo = blo;
        }

        // ================= segment argmin over (start, rank, op) ==============================
        uint32_t mh = khi, ml = klo;
#pragma unroll
        for (int off = 1; off < SEG; off <<= 1) {
            uint32_t oh = __shfl_xor_sync(0xffffffffu, mh, off);
            uint32_t ol = __shfl_xor_sync(0xffffffffu, ml, off);
            if (oh < mh || (oh == mh && ol < ml)) { mh = oh; ml = ol; }
        }
        const bool seg_ovf = (__ballot_sync(0xffffffffu, ovf) & segmask) != 0u;

        if (alive) {
            if (seg_ovf) {
                // hand the candidate to the global-state variant
                if (i == 0) {
                    int at = atomicAdd(p.ovf_count, 1);
                    p.ovf_list[at] = (int32_t)cand;
                }
                alive = false;
            } else if (mh == KEY_NONE) {
                // ===== finished or deadlocked =====
                unsigned rem = __ballot_sync(segmask, has_stage && pos < L) & segmask;
                if (rem == 0u) {
                    win_fold(INT_MAX);
                    int hi, lo_;
                    if (p.post) {
                        hi = has_stage ? last_w - first_f : 0;
                        lo_ = 0;
                    } else {
                        hi = has_stage ? sfree : 0;
                        lo_ = has_stage ? first_start : INT_MAX;
                    }
                    for (int off = 1; off < SEG; off <<= 1) {
                        hi = max(hi, __shfl_xor_sync(segmask, hi, off));
                        lo_ = min(lo_, __shfl_xor_sync(segmask, lo_, off));
                    }
                    const long long span = (long long)hi - (long long)lo_;
                    if (p.peak && has_stage) p.peak[(size_t)cand * P + i] = (long long)peak * p.unit;
                    if (i == 0) {
                        put_result(FLAG_FEASIBLE, span, 0u);
                        if (MOVES && p.best_key) {
                            long long key = (span << 32) | (long long)(uint32_t)(p.first_index + cand);
                            if (key < *(volatile long long *)p.best_key) atomicMin(p.best_key, key);
                        }
                    }
                } else {
                    if (i == 0) put_result(FLAG_DEADLOCK, -1LL, rem >> (seg * SEG));
                    if (p.peak && has_stage) p.peak[(size_t)cand * P + i] = -1;
                }
                alive = false;
            } else {
                // ===== commit the winner =====
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
                        win_insert(end, val_of(j, k));
                        sfree = end;
                        ++pos;
                        head = nxt;
                        nxt = fetch(pos + 1);
                        if (first_start == INT_MAX) first_start = t;
                        if (k == KIND_F) {
                            A_i[j] = ((uint32_t)end << 2) | 1u;
                            if (first_f == INT_MAX) first_f = t;
                            if (derived && ((offm_i[j >> 5] >> (j & 31)) & 1u)) poff_i[j >> 5] |= 1u << (j & 31);
                        } else if (k == KIND_B) {
                            A_i[j] = ((uint32_t)end << 2) | 2u;
                        } else {
                            last_w = end;
                        }
                    }
                    dirty = dirty || i == w || (k == KIND_F && i == w + 1) || (k == KIND_B && i == w - 1);
                } else {
                    const int end = t + p.toff;
                    const int wch = __ldg(&p.chan[w]);
                    if (has_stage && chan_i == wch) {
                        cfree = end;
                        dirty = true;
                        if (!derived) {
                            ++cpos;
                            chead = cnext;
                            cnext = fetch_chan(cpos + 1);
                        }
                    }
                    if (i == w) {
                        const V g = val_of(j, 3);
                        const uint32_t bit = 1u << (j & 31);
                        if (rank == RANK_OFFLOAD) {
                            X_i[j] = ((uint32_t)end << 2) | 1u;
                            win_insert(end, -g);
                            if (derived) { poff_i[j >> 5] &= ~bit; prel_i[j >> 5] |= bit; }
                        } else {
                            X_i[j] = ((uint32_t)end << 2) | 2u;
                            win_insert(t, g);
                            if (derived) prel_i[j >> 5] &= ~bit;
                        }
                    }
                }
            }
        }
        __syncwarp();
    }
}

}  // namespace ps
