// ps_bound.cu — batched branch-and-bound node lower bound.
//
// Restates solver._Search._bound (solver.py:352-383) with _chain_ends (solver.py:321-350) for a
// batch of B&B nodes at once: a parallel frontier is bounded in one launch instead of one Python
// call per node.  A node is (clock t, stage free times, committed compute starts); its bound is
//   non-post: max(committed ends, max(sfree_i, t) + remaining work_i, chain ends) - min start,
//   post:     max over stages of the stage's span bound,
// where chain ends are the earliest ends of every op along its F chain down the stages, B chain up
// the stages and W after its B, each floored by max(t, sfree_i) (stage queueing ignored).
//
// One warp per node, lanes over microbatches (chains of different microbatches are independent);
// per-stage sums and extrema are warp reductions.  Integer work, HBM-bound on the start tables.
#include <cuda_runtime.h>
#include <stdint.h>
#include <climits>

#include "../../include/pipesched_b200.h"

namespace {

struct BoundParams {
    int P, m, uniform, post, comm;
    const int32_t *proc;          // instance table: [P or P*m][3]
    int64_t N;
    const int32_t *clock;         // [N]
    const int32_t *sfree;         // [N][P]
    const int32_t *start;         // [N][P][m][3], -1 = not committed
    int64_t *lb;                  // [N]
};

__device__ __forceinline__ long long warp_sum(long long v) {
#pragma unroll
    for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}
__device__ __forceinline__ long long warp_max(long long v) {
#pragma unroll
    for (int o = 16; o; o >>= 1) v = max(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}
__device__ __forceinline__ long long warp_min(long long v) {
#pragma unroll
    for (int o = 16; o; o >>= 1) v = min(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}

__global__ void __launch_bounds__(128) bound_kernel(const BoundParams b) {
    const int lane = threadIdx.x & 31;
    const long long warp = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const long long nwarps = ((long long)gridDim.x * blockDim.x) >> 5;
    const int P = b.P, m = b.m;
    auto pt = [&](int i, int j, int k) -> long long {
        return __ldg(&b.proc[((b.uniform ? i : i * m + j)) * 3 + k]);
    };
    for (long long n = warp; n < b.N; n += nwarps) {
        const long long t = __ldg(&b.clock[n]);
        const int32_t *sf = b.sfree + n * P;
        const int32_t *st = b.start + n * (long long)P * m * 3;
        auto S = [&](int i, int j, int k) -> long long { return __ldg(&st[((long long)i * m + j) * 3 + k]); };
        long long res;
        if (b.post) {
            long long worst = 0;                                         // solver.py:354-369
            for (int i = 0; i < P; ++i) {
                long long rem = 0, first_f = LLONG_MAX, last_w = LLONG_MIN;
                int have_f = 0;
                for (int j = lane; j < m; j += 32)
                    for (int k = 0; k < 3; ++k) {
                        const long long s = S(i, j, k);
                        if (s < 0) { rem += pt(i, j, k); continue; }
                        if (k == 0) { have_f = 1; first_f = min(first_f, s); }
                        if (k == 2) last_w = max(last_w, s + pt(i, j, 2));
                    }
                rem = warp_sum(rem);
                first_f = warp_min(first_f);
                last_w = warp_max(last_w);
                have_f = __any_sync(0xffffffffu, have_f);
                const long long fl = max((long long)__ldg(&sf[i]), t);
                const long long v = rem == 0 ? last_w - first_f : (have_f ? fl + rem - first_f : rem);
                worst = max(worst, v);
            }
            res = worst;
        } else {
            long long lb = 0, min_start = LLONG_MAX;                       // solver.py:370-383
            int any = 0;
            for (int i = 0; i < P; ++i) {
                const long long fl = max((long long)__ldg(&sf[i]), t);
                long long rem = 0;
                for (int j = lane; j < m; j += 32)
                    for (int k = 0; k < 3; ++k) {
                        const long long s = S(i, j, k);
                        if (s < 0) rem += pt(i, j, k);
                        else { any = 1; lb = max(lb, s + pt(i, j, k)); min_start = min(min_start, s); }
                    }
                rem = warp_sum(rem);
                if (rem) lb = max(lb, fl + rem);
            }
            // _chain_ends, one microbatch per lane at a time: F down the stages, B up with W after B
            long long ef[32];
            for (int j = lane; j < m; j += 32) {
                for (int i = 0; i < P; ++i) {
                    const long long s = S(i, j, 0);
                    long long e;
                    if (s >= 0) e = s + pt(i, j, 0);
                    else {
                        long long lo = max((long long)__ldg(&sf[i]), t);
                        if (i > 0) lo = max(lo, ef[i - 1] + b.comm);
                        e = lo + pt(i, j, 0);
                    }
                    ef[i] = e;
                    lb = max(lb, e);
                }
                long long eb_up = 0;
                for (int i = P - 1; i >= 0; --i) {
                    const long long fl = max((long long)__ldg(&sf[i]), t);
                    const long long sb = S(i, j, 1);
                    long long eb;
                    if (sb >= 0) eb = sb + pt(i, j, 1);
                    else {
                        long long lo = max(fl, ef[i]);
                        if (i < P - 1) lo = max(lo, eb_up + b.comm);
                        eb = lo + pt(i, j, 1);
                    }
                    const long long sw = S(i, j, 2);
                    const long long ew = sw >= 0 ? sw + pt(i, j, 2) : max(fl, eb) + pt(i, j, 2);
                    lb = max(lb, max(eb, ew));
                    eb_up = eb;
                }
            }
            lb = warp_max(lb);
            min_start = warp_min(min_start);
            any = __any_sync(0xffffffffu, any);
            res = any ? lb - min_start : lb;
        }
        if (lane == 0) b.lb[n] = res;
    }
}

}  // namespace

// Exposed to ps_abi.cu (same library).
extern "C" cudaError_t ps_bound_launch(int P, int m, int uniform, int post, int comm, const int32_t *proc, int64_t N,
                            const int32_t *clock, const int32_t *sfree, const int32_t *start, int64_t *lb,
                            int num_sms, cudaStream_t s) {
    BoundParams b;
    b.P = P; b.m = m; b.uniform = uniform; b.post = post; b.comm = comm; b.proc = proc;
    b.N = N; b.clock = clock; b.sfree = sfree; b.start = start; b.lb = lb;
    const long long warps = N;
    int grid = (int)((warps * 32 + 127) / 128);
    const int cap = 16 * num_sms;
    if (grid > cap) grid = cap;
    if (grid < 1) grid = 1;
    bound_kernel<<<grid, 128, 0, s>>>(b);
    return cudaGetLastError();
}
