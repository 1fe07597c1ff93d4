// ps_literal.cu — the reference's run_order replayed literally, for stage rows that are not
// permutations of the stage's ops.
//
// listsched.run_order (listsched.py:167-269) does not validate its input: a row may repeat an op
// (the repeat is committed again: its end time is overwritten, its memory delta added again,
// its stage position advances) or be shorter than 3m (it simply ends).  Such a row leaves some
// op of its stage uncommitted, so the loop `while len(done) < total ...` can never finish and the
// run ends in OrderInfeasible with the rows not yet exhausted as `stages` (listsched.py:248-252).
// The evaluator kernel (ps_eval.cuh) assumes permutations and flags these candidates
// PS_FLAG_MALFORMED; this pass re-runs exactly those, one thread each, with the reference's own
// data structures restated over dense arrays (sorted ledger with insertion, earliest_fit walking
// its breakpoints, requested-set refresh), and replaces the flag with the reference's outcome:
// PS_FLAG_DEADLOCK and the blocked-stage mask.  A candidate whose op codes name no op of the
// stage (microbatch >= m, kind 3) or whose offload bits name a non-offloadable F stays MALFORMED
// (the reference raises KeyError or worse there).
//
// The same pass finishes, in 64-bit time, every candidate the evaluator ended with PS_FLAG_RANGE
// (an event time reached 2^29 quanta, the limit of its packed 32-bit end-time words): makespan,
// bubble, STRICT peaks and the commit-ordered trace as the reference computes them
// (schedule.py:168-237, cli.py:115), so instances with long horizons get exact answers for every
// candidate (a trace time that does not fit the int32 trace output keeps PS_FLAG_RANGE).
//
// Rare by construction (malformed input, very long schedules), so the simplest correct mapping:
// one thread per candidate, state in a global scratch slot, a few thousand slots at most.
#include <cuda_runtime.h>
#include <stdint.h>
#include <climits>
#include "ps_eval.cuh"
#include "ps_literal.h"

namespace ps {
namespace {

constexpr int64_t T_NONE = INT64_MIN;
constexpr uint32_t ROW_END = 0xFFFFu;

struct Pt {
    int64_t t, d;
};

template <typename V>
__device__ __forceinline__ int64_t val(const void *base, int idx) {
    return (int64_t)reinterpret_cast<const V *>(base)[idx];
}

// _MemLedger.earliest_fit (listsched.py:62-100): smallest t >= lo with usage + delta <= limit at
// every time >= t + lag, walking forward over breakpoints; T_NONE when none.
__device__ int64_t earliest_fit(const Pt *pts, int n, int64_t limit, int64_t lo, int64_t delta, int64_t lag) {
    if (delta <= 0) return lo;
    int64_t t = lo;
    for (;;) {
        // worst usage over [t + lag, inf): the plateau entering t + lag and every later breakpoint
        const int64_t T = t + lag;
        int64_t run = 0, cur = 0, later = INT64_MIN;
        bool any_later = false;
        for (int k = 0; k < n;) {
            const int64_t bt = pts[k].t;
            while (k < n && pts[k].t == bt) run += pts[k++].d;          // merged same-time deltas
            if (bt <= T) cur = run;
            else { any_later = true; later = later > run ? later : run; }
        }
        const int64_t worst = any_later ? (cur > later ? cur : later) : cur;
        if (worst + delta <= limit) return t;
        int64_t nxt = T_NONE;
        for (int k = 0; k < n; ++k)
            if (pts[k].t > T) { nxt = pts[k].t; break; }
        if (nxt == T_NONE) return T_NONE;
        t = nxt - lag;
    }
}

__device__ void ledger_add(Pt *pts, int *n, int64_t t, int64_t d) {
    // insort of (t, d): after every point that compares <= (t, d)
    int k = *n;
    while (k > 0 && (pts[k - 1].t > t || (pts[k - 1].t == t && pts[k - 1].d > d))) {
        pts[k] = pts[k - 1];
        --k;
    }
    pts[k].t = t;
    pts[k].d = d;
    ++*n;
}

// The candidates this pass replays (flagged malformed or out of range), compacted by one thread
// per candidate: the replay threads then walk only those (usually none).
__global__ void collect_kernel(const uint32_t *flags, int64_t N, int32_t *list) {
    const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= N) return;
    const uint32_t f = flags[c];
    if (f == FLAG_MALFORMED || f == FLAG_RANGE) list[1 + atomicAdd(list, 1)] = (int32_t)c;
}

template <typename V>
__global__ void literal_kernel(const EvalParams p, int64_t *scratch, int slot_words, int slots,
                               const int32_t *list) {
    const int P = p.P, m = p.m, G = p.G, L = p.L;
    const int tid = blockIdx.x * blockDim.x + threadIdx.x;
    if (tid >= slots) return;
    int64_t *base = scratch + (size_t)tid * slot_words;
    // slot layout (int64 words)
    int64_t *done = base;                          // [P*m*3] end time or -1
    int64_t *off_end = done + (size_t)P * m * 3;   // [P*m]
    int64_t *rel_end = off_end + (size_t)P * m;    // [P*m]
    int64_t *sfree = rel_end + (size_t)P * m;      // [P]
    int64_t *cfree = sfree + P;                    // [G]
    int64_t *first_start = cfree + G;              // [P] start of the stage's first compute
    // earliest_fit answers, cached until the stage's ledger grows (its point count is its version):
    // the F head's per stage (keyed by position and floor), each reload's per activation (by floor)
    int64_t *fc_lo = first_start + P, *fc_res = fc_lo + P;              // [P]
    int64_t *rc_lo = fc_res + P, *rc_res = rc_lo + (size_t)P * m;       // [P*m]
    const int cap = 5 * m + 8;                     // ledger points per stage: <= len(row) + 2m
    Pt *pts = reinterpret_cast<Pt *>(rc_res + (size_t)P * m);   // [P][cap]
    int32_t *ints = reinterpret_cast<int32_t *>(pts + (size_t)P * cap);
    int32_t *npts = ints;                          // [P]
    int32_t *pos = npts + P;                       // [P]
    int32_t *len = pos + P;                        // [P]
    int32_t *cpos = len + P;                       // [G]
    int32_t *fc_n = cpos + G, *fc_pos = fc_n + P;  // [P] cache keys: ledger points, head position
    int32_t *rc_n = fc_pos + P;                    // [P*m]
    int32_t *pend = rc_n + (size_t)P * m;          // [P*m] (derived mode) requested, not yet reloaded
    uint8_t *req = reinterpret_cast<uint8_t *>(pend + (size_t)P * m);   // [P*m] bit0 offload, bit1 reload requested
    const int mwords = (P * m + 31) / 32;
    const int n_list = *list;
    for (int k = tid; k < n_list; k += slots) {
        const int64_t c = list[1 + k];
        const uint32_t flag_in = p.flags[c];
        if (flag_in != FLAG_MALFORMED && flag_in != FLAG_RANGE) continue;
        // ---- op codes and offload bits must name ops of the instance --------------------------
        bool bad = false;
        auto code_at = [&](int i, int q) -> uint32_t {
            const size_t idx = ((size_t)c * P + i) * p.stride + q;
            if (p.order_u8) {
                const uint32_t b = reinterpret_cast<const uint8_t *>(p.orders)[idx];
                return b == 0xFFu ? ROW_END : b;
            }
            return reinterpret_cast<const uint16_t *>(p.orders)[idx];
        };
        for (int i = 0; i < P && !bad; ++i) {
            len[i] = L;
            for (int q = 0; q < L; ++q) {
                const uint32_t op = code_at(i, q);
                if (op == ROW_END) { len[i] = q; break; }
                if ((op >> 2) >= (uint32_t)m || (op & 3u) > 2u) { bad = true; break; }
            }
        }
        int n_off = 0;
        auto offloaded = [&](int x) -> bool { return (p.masks[(size_t)c * mwords + (x >> 5)] >> (x & 31)) & 1u; };
        for (int x = 0; x < P * m && !bad; ++x)
            if (offloaded(x)) {
                if (val<V>(p.vals, (p.uniform ? x / m : x) * 4 + 3) <= 0) bad = true;
                ++n_off;
            }
        if (bad) continue;                                  // stays PS_FLAG_MALFORMED
        if (p.chorders) {
            // explicit channel orders must name offloaded ops served by their channel
            for (int g = 0; g < G && !bad; ++g)
                for (int q = 0; q < p.chan_stride; ++q) {
                    const uint32_t e = p.chorders[((size_t)c * G + g) * p.chan_stride + q];
                    if (e == NO_CHAN) break;
                    const int i = (int)((e >> 16) & 0x7FFFu), j = (int)(e & 0xFFFFu);
                    if (i >= P || j >= m || !offloaded(i * m + j) || p.chan[i] != g) { bad = true; break; }
                }
            if (bad) continue;
        }
        // ---- run_order, literally (listsched.py:170-267) ------------------------------------
        for (int k = 0; k < P * m * 3; ++k) done[k] = -1;
        for (int k = 0; k < P * m; ++k) { off_end[k] = rel_end[k] = -1; req[k] = 0; }
        for (int i = 0; i < P; ++i) { sfree[i] = 0; npts[i] = 0; pos[i] = 0; fc_n[i] = -1; }
        for (int k = 0; k < P * m; ++k) rc_n[k] = -1;
        for (int g = 0; g < G; ++g) { cfree[g] = 0; cpos[g] = 0; }
        const bool derived = p.chorders == nullptr;
        const long long total = 3LL * P * m, total_tr = 2LL * n_off;
        long long n_done = 0, n_tr = 0;
        int n_pend = 0;
        auto proc = [&](int i, int j, int k) -> int64_t { return p.proc[((p.uniform ? i : i * m + j)) * 3 + k]; };
        auto vrow = [&](int i, int j, int k) -> int64_t { return val<V>(p.vals, (p.uniform ? i : i * m + j) * 4 + k); };
        auto D = [&](int i, int j, int k) -> int64_t & { return done[((size_t)i * m + j) * 3 + k]; };
        uint32_t blocked = 0u;
        bool deadlock = false;
        long long ecount = 0;
        bool trace_ovf = false;
        int64_t lo_start = INT64_MAX, hi_end = INT64_MIN;
        for (int i = 0; i < P; ++i) first_start[i] = INT64_MAX;
        while (n_done < total || n_tr < total_tr) {
            // (the derived-mode pending list is the requested set minus what was committed:
            // selection below is by the minimum key, so the list order never matters)
            int64_t bt = 0;
            int brank = -1, bi = 0, bj = 0, bk = 0, bg = 0;
            auto better = [&](int64_t t, int rank, int i, int j, int k) -> bool {
                if (brank < 0) return true;
                if (t != bt) return t < bt;
                if (rank != brank) return rank < brank;
                if (i != bi) return i < bi;
                if (j != bj) return j < bj;
                return k < bk;
            };
            for (int i = 0; i < P; ++i) {                          // stage heads (listsched.py:217-232)
                if (pos[i] >= len[i]) continue;
                const uint32_t op = code_at(i, pos[i]);
                const int j = (int)(op >> 2), k = (int)(op & 3u);
                // _compute_ready (listsched.py:114-145)
                int64_t fl = 0;
                bool ready = true;
                if (k == KIND_F) {
                    if (i > 0) { const int64_t u = D(i - 1, j, 0); if (u < 0) ready = false; else fl = max(fl, u + p.comm); }
                } else if (k == KIND_B) {
                    const int64_t f = D(i, j, 0);
                    if (f < 0) ready = false; else fl = max(fl, f);
                    if (ready && i < P - 1) { const int64_t d = D(i + 1, j, 1); if (d < 0) ready = false; else fl = max(fl, d + p.comm); }
                    if (ready && offloaded(i * m + j)) { const int64_t r = rel_end[i * m + j]; if (r < 0) ready = false; else fl = max(fl, r); }
                } else {
                    const int64_t b = D(i, j, 1);
                    if (b < 0) ready = false; else fl = max(fl, b);
                }
                if (!ready) continue;
                int64_t lo = max(fl, sfree[i]);
                if (k == KIND_F) {
                    if (fc_n[i] != npts[i] || fc_pos[i] != pos[i] || fc_lo[i] != lo) {
                        fc_n[i] = npts[i];
                        fc_pos[i] = pos[i];
                        fc_lo[i] = lo;
                        fc_res[i] = earliest_fit(pts + (size_t)i * cap, npts[i], val<V>(p.limit, i), lo, vrow(i, j, 0), proc(i, j, 0));
                    }
                    lo = fc_res[i];
                    if (lo == T_NONE) continue;
                }
                if (better(lo, RANK_COMPUTE, i, j, k)) { bt = lo; brank = RANK_COMPUTE; bi = i; bj = j; bk = k; }
            }
            auto transfer = [&](int g, int x, bool reload) {       // transfer_candidate (186-204)
                const int64_t floor_t = reload ? off_end[x] : D(x / m, x % m, 0);
                if (floor_t < 0) return;
                int64_t lo = max(floor_t, cfree[g]);
                const int i = x / m, j = x % m;
                if (reload) {
                    if (rc_n[x] != npts[i] || rc_lo[x] != lo) {
                        rc_n[x] = npts[i];
                        rc_lo[x] = lo;
                        rc_res[x] = earliest_fit(pts + (size_t)i * cap, npts[i], val<V>(p.limit, i), lo, vrow(i, j, 3), 0);
                    }
                    lo = rc_res[x];
                    if (lo == T_NONE) return;
                }
                const int rank = reload ? RANK_RELOAD : RANK_OFFLOAD;
                if (better(lo, rank, i, j, 0)) { bt = lo; brank = rank; bi = i; bj = j; bk = 0; bg = g; }
            };
            if (derived) {
                // refresh (listsched.py:207-214): a request appears once its producer commits (the
                // commits below keep the requested-not-reloaded activations in `pend`; selection is
                // by the minimum key, so the list order never matters)
                for (int q = 0; q < n_pend; ++q) {
                    const int x = pend[q];
                    const int g = p.chan[x / m];
                    if ((req[x] & 1) && !(req[x] & 4)) transfer(g, x, false);      // bit 2: offload committed
                    if ((req[x] & 2) && !(req[x] & 8)) transfer(g, x, true);       // bit 3: reload committed
                }
            } else {
                for (int g = 0; g < G; ++g) {
                    if (cpos[g] >= p.chan_stride) continue;
                    const uint32_t e = p.chorders[((size_t)c * G + g) * p.chan_stride + cpos[g]];
                    if (e == NO_CHAN) continue;
                    transfer(g, (int)((e >> 16) & 0x7FFFu) * m + (int)(e & 0xFFFFu), (e >> 31) != 0u);
                }
            }
            if (brank < 0) {                                        // OrderInfeasible (248-252)
                for (int i = 0; i < P; ++i)
                    if (pos[i] < len[i]) blocked |= 1u << i;
                deadlock = true;
                break;
            }
            if (p.tcode) {                                          // commit-ordered trace
                if (bt > INT_MAX) trace_ovf = true;
                else if (ecount < p.tstride) {
                    p.tcode[(size_t)c * p.tstride + ecount] = ((uint32_t)brank << 30) | ((uint32_t)bi << 24) |
                                                              ((uint32_t)bj << 2) | (uint32_t)bk;
                    p.tstart[(size_t)c * p.tstride + ecount] = (int32_t)bt;
                }
            }
            ++ecount;
            if (brank == RANK_COMPUTE) {                            // _commit_compute (148-152)
                const int64_t end = bt + proc(bi, bj, bk);
                lo_start = min(lo_start, bt);
                hi_end = max(hi_end, end);
                if (first_start[bi] == INT64_MAX) first_start[bi] = bt;
                if (D(bi, bj, bk) < 0) ++n_done;                    // len(done) counts distinct ops
                D(bi, bj, bk) = end;
                if (derived && bk == KIND_F && offloaded(bi * m + bj) && !(req[bi * m + bj] & 1)) {
                    req[bi * m + bj] |= 1;                          // offload requested
                    pend[n_pend++] = bi * m + bj;
                }
                ledger_add(pts + (size_t)bi * cap, &npts[bi], end, vrow(bi, bj, bk));
                ++pos[bi];
                sfree[bi] = end;
            } else {                                                // _commit_transfer (155-164)
                const int x = bi * m + bj;
                const int64_t end = bt + p.toff, gamma = vrow(bi, bj, 3);
                if (brank == RANK_OFFLOAD) {
                    off_end[x] = end;
                    ledger_add(pts + (size_t)bi * cap, &npts[bi], end, -gamma);
                    req[x] |= 4 | 2;                                // committed; reload requested
                } else {
                    rel_end[x] = end;
                    ledger_add(pts + (size_t)bi * cap, &npts[bi], bt, gamma);
                    req[x] |= 8;
                    if (derived)
                        for (int q = 0; q < n_pend; ++q)
                            if (pend[q] == x) { pend[q] = pend[--n_pend]; break; }
                }
                cfree[bg] = end;
                if (!derived) ++cpos[bg];
                ++n_tr;
            }
        }
        if (p.events_total) atomicAdd(p.events_total, (unsigned long long)ecount);
        if (!deadlock) {
            // (rows that miss an op cannot get here; a range candidate finishes)
            if (flag_in != FLAG_RANGE || trace_ovf) continue;
            // makespan (schedule.py:168-183): global compute span, or the worst per-stage span
            int64_t span;
            if (p.post) {
                span = 0;
                for (int i = 0; i < P; ++i) span = max(span, sfree[i] - first_start[i]);
            } else {
                span = hi_end - lo_start;
            }
            if (p.events_total) atomicAdd(p.events_total + 1, (unsigned long long)(total + total_tr));
            p.flags[c] = FLAG_FEASIBLE;
            if (p.makespan) p.makespan[c] = span;
            if (p.bubble)
                p.bubble[c] = span > 0 ? 1.0 - (double)p.busy / ((double)P * (double)span)
                                       : __longlong_as_double(0x7ff8000000000000LL);
            if (p.blocked) p.blocked[c] = 0u;
            if (p.peak)
                for (int i = 0; i < P; ++i) {
                    // STRICT memory_trace peak (schedule.py:207-237): prefix sums of same-time merged deltas
                    const Pt *q = pts + (size_t)i * cap;
                    int64_t run = 0, pk = 0;
                    for (int k = 0; k < npts[i];) {
                        const int64_t t0 = q[k].t;
                        while (k < npts[i] && q[k].t == t0) run += q[k++].d;
                        pk = max(pk, run);
                    }
                    p.peak[(size_t)c * P + i] = pk * p.unit;
                }
            continue;
        }
        p.flags[c] = FLAG_DEADLOCK;
        if (p.makespan) p.makespan[c] = -1;
        if (p.bubble) p.bubble[c] = __longlong_as_double(0x7ff8000000000000LL);
        if (p.blocked) p.blocked[c] = blocked;
        if (p.peak)
            for (int i = 0; i < P; ++i) p.peak[(size_t)c * P + i] = -1;
    }
}

}  // namespace

size_t literal_slot_bytes(int P, int m, int G) {
    const size_t words = (size_t)P * m * 3 + 4 * (size_t)P * m + 4 * P + G;
    const size_t pts = (size_t)P * (5 * m + 8) * sizeof(Pt);
    const size_t ints = (size_t)(5 * P + G) * 4 + 2 * (size_t)P * m * 4 + (size_t)P * m;
    return (words * 8 + pts + ints + 15) & ~(size_t)15;
}

cudaError_t literal_launch(const EvalParams &p, bool v64, int64_t *scratch, int slots, cudaStream_t s) {
    const int slot_words = (int)(literal_slot_bytes(p.P, p.m, p.G) / 8);
    int32_t *list = nullptr;
    cudaError_t e = cudaMallocAsync((void **)&list, (size_t)(p.N + 1) * sizeof(int32_t), s);
    if (e != cudaSuccess) return e;
    e = cudaMemsetAsync(list, 0, sizeof(int32_t), s);
    if (e != cudaSuccess) return e;
    collect_kernel<<<(unsigned)((p.N + 255) / 256), 256, 0, s>>>(p.flags, p.N, list);
    const int block = 64, grid = (slots + block - 1) / block;
    if (v64) literal_kernel<long long><<<grid, block, 0, s>>>(p, scratch, slot_words, slots, list);
    else literal_kernel<int><<<grid, block, 0, s>>>(p, scratch, slot_words, slots, list);
    e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    return cudaFreeAsync(list, s);
}

}  // namespace ps
