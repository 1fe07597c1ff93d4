// ps_abi.cu — C ABI (include/pipesched_b200.h): instance tables, launch planning, search kernels.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>
#include <nvtx3/nvToolsExt.h>
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_select.cuh>
#include <climits>
#include <stdarg.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <algorithm>
#include <map>
#include <mutex>
#include <new>
#include <string>
#include <vector>

#include "../../include/pipesched_b200.h"
#include "ps_launch.h"
#include "ps_literal.h"

using namespace ps;

namespace {
// NVTX ranges around every entry point (header-only NVTX3: free unless a profiler is attached),
// so nsys/ncu timelines show rounds, batches and recordings by name.
struct NvtxRange {
    explicit NvtxRange(const char *name) { nvtxRangePushA(name); }
    NvtxRange(const char *fmt, unsigned long long v) {
        char buf[96];
        snprintf(buf, sizeof buf, fmt, v);
        nvtxRangePushA(buf);
    }
    ~NvtxRange() { nvtxRangePop(); }
};
}  // namespace

struct ps_instance {
    int device;
    int num_sms;
    int max_smem_optin;
    int P, m, G, L, MW, stride, mask_words;
    int comm, toff, post, uniform, any_off;
    int time_safe;            // see EvalParams::time_safe
    int64_t busy, unit;
    bool v64;
    int32_t *d_proc;
    void *d_vals;
    void *d_limit;
    int32_t *d_chan;
    std::vector<uint8_t> h_offloadable;   // [P][m]
    // occupancy answers per launch shape (the query costs microseconds per call otherwise)
    mutable std::mutex occ_mu;
    mutable std::map<uint64_t, int> occ_cache;
};

struct ps_base {
    const ps_instance *inst;
    int K, cand_words, ck_words, ck_interval, ck_max;
    mutable int max_window;     // widest live ledger window the base needed (-1: unknown / unusable)
    // the recording's info reaches the host asynchronously (no stream sync per recording)
    int32_t *h_info = nullptr;  // pinned [8]
    cudaEvent_t info_ev = nullptr;
    mutable bool info_pending = false;
    uint32_t *ck;       // [ck_max][ck_words]
    uint32_t *cstep;    // [P][L]
    uint32_t *fstep;    // [P][m]
    int32_t *info;      // [4]
    int64_t *res;       // [2 + 3P]
    uint16_t *orders;   // [P][stride]
    uint32_t *mask;     // [mask_words]
    uint16_t *prev_orders;   // the previously recorded base (a re-recording resumes from its checkpoints)
    uint32_t *prev_mask;
    // explicit channel orders (ps_base_record_explicit): the base's [G][chan_stride] rows, the
    // previous base's, and the compute index at which each channel position committed
    int chan_stride = 0;     // of the current recording (0: derived channel mode)
    int rec_stride = -1;     // mode of the last recording (-1: none)
    int cap_stride = 0;
    uint32_t *chorders = nullptr, *prev_chorders = nullptr, *chstep = nullptr;
};

namespace {

thread_local std::string g_last_error;

int fail(int code, const char *fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    g_last_error = buf;
    return code;
}

int cuda_fail(cudaError_t e, const char *what) {
    return fail(PS_ERR_CUDA, "%s: %s", what, cudaGetErrorString(e));
}

#define PS_CUDA(call)                                            \
    do {                                                         \
        cudaError_t e_ = (call);                                 \
        if (e_ != cudaSuccess) return cuda_fail(e_, #call);      \
    } while (0)

// Make `dev` current for the duration of a call and restore the caller's device afterwards.
struct DeviceGuard {
    int prev = -1;
    bool ok = true;
    explicit DeviceGuard(int dev) {
        if (cudaGetDevice(&prev) != cudaSuccess) { ok = false; return; }
        if (prev != dev && cudaSetDevice(dev) != cudaSuccess) ok = false;
    }
    ~DeviceGuard() {
        int cur;
        if (prev >= 0 && cudaGetDevice(&cur) == cudaSuccess && cur != prev) cudaSetDevice(prev);
    }
};

int64_t gcd64(int64_t a, int64_t b) {
    if (a < 0) a = -a;
    if (b < 0) b = -b;
    while (b) {
        int64_t t = a % b;
        a = b;
        b = t;
    }
    return a;
}

int next_pow2(int x) {
    int p = 1;
    while (p < x) p <<= 1;
    return p;
}

struct Plan {
    int K, warps;
    bool gstate;
    bool win_smem;      // global state: the ledger windows in shared memory
    int cand_words, inc_words;
    LaunchCfg cfg;
    size_t scratch_bytes;
};

// Per-candidate state words: ledger windows, end-time rows and bitsets, then (materialised
// candidates, order_bytes > 0) the staged stage orders.
int words_per_candidate(const ps_instance *I, int K, int order_bytes = 0) {
    int vw = I->v64 ? 2 : 1;
    int nz = 2 * I->P * I->m + 3 * I->P * I->MW;
    int w = I->P * 2 * K * (vw + 1) + ((nz + 3) & ~3) + I->P * I->stride * order_bytes / 4;   // rows 16-byte aligned
    return (w + 3) & ~3;
}

int incumbent_words(const ps_instance *I, bool moves) {
    if (!moves) return 0;
    int w = I->P * I->stride / 2 + I->mask_words;
    return (w + 3) & ~3;
}

cudaError_t occupancy(bool v64, bool moves, Variant v, int block, size_t smem, int *n) {
    if (v64) return moves ? eval_occupancy<long long, true>(v, block, smem, n) : eval_occupancy<long long, false>(v, block, smem, n);
    return moves ? eval_occupancy<int, true>(v, block, smem, n) : eval_occupancy<int, false>(v, block, smem, n);
}

int env_int(const char *name, int dflt) {
    const char *v = getenv(name);
    return v && *v ? atoi(v) : dflt;
}

// Global-state kernels with nonzero-word masks over the pending-transfer sets: for stages with
// many bitset words (config 5, MW = 8: 15.9 vs 17.5 ms per round); with few (config 4, MW = 4) the
// plain scan is faster (4.29 vs 4.55 ms).
bool wmask_shape(int MW) {
    static const int on = env_int("PS_WMASK", 1);
    return on && MW >= 6 && MW <= 16;
}

// Materialised shared-memory passes with no recorded base run the full-simulation build (no
// checkpoint code, 7 blocks per SM): no-base batches 55.4 -> 49.7 ms at config 3 (r02 A/B).
// With global state (GS 4, one-warp blocks at 80 registers, up to 24 per SM) it pays only for
// states of up to ~40 KB: config 4 (33 KB with its staged rows) 445 -> 342 ms per 65,536 full
// simulations; config 5 (118 KB) was slower at 16 or 24 blocks per SM (1.23-1.39 vs 1.13 s) and
// keeps the general build.
bool nobase_build(bool moves, bool gstate, bool record, bool has_base, int cand_words = 0) {
    static const int on = env_int("PS_NOBASE_BUILD", 1);
    if (gstate && (int64_t)cand_words * 4 > env_int("PS_GNB_MAX_BYTES", 40960)) return false;
    return on && !moves && !record && !has_base;
}

cudaError_t launch(bool v64, bool moves, bool gstate, const EvalParams &p, LaunchCfg c, cudaStream_t s,
                   bool record = false) {
    Variant v;
    v.gstate = gstate;
    v.record = record;
    v.derived = p.chorders == nullptr;
    v.uni = p.uniform != 0;
    v.wmask = gstate && wmask_shape(p.MW);
    v.nobase = nobase_build(moves, gstate, record, p.ck != nullptr, p.cand_words);
    if (v64) return moves ? eval_launch<long long, true>(v, p, c, s) : eval_launch<long long, false>(v, p, c, s);
    return moves ? eval_launch<int, true>(v, p, c, s) : eval_launch<int, false>(v, p, c, s);
}


// Shared-memory plan for the main pass: one candidate per warp, ledger window K (12 by default, or
// the whole 5m ledger when that is smaller and cannot overflow), as many warps per block as fit;
// state moves to global memory only when a single warp's state does not fit.
int window_size(const ps_instance *I) { return std::min(std::max(4, env_int("PS_WINDOW", 16)), 5 * I->m); }

// One evaluation pass with ledger window K: one candidate per warp, as many warps per block as fit
// in shared memory; the state moves to global memory only when a single warp's does not fit.
// `N` bounds the grid (a worklist pass may receive fewer candidates, never more).
int plan_pass(const ps_instance *I, bool moves, int K, int64_t N, Plan *pl, int order_bytes = 2,
              bool has_base = true) {
    K = (K + 1) & ~1;            // even: the state words after the windows start on a 16-byte boundary
    pl->K = K;
    pl->cand_words = words_per_candidate(I, K, moves ? 0 : order_bytes);
    pl->inc_words = incumbent_words(I, moves);
    pl->gstate = true;
    pl->win_smem = false;
    pl->warps = 4;
    const int max_warps = std::max(1, std::min(4, env_int("PS_WARPS_PER_BLOCK", 4)));
    const bool force_g = env_int("PS_FORCE_GSTATE", 0) != 0;     // (experiments)
    for (int w : {4, 2, 1}) {
        if (w > max_warps || force_g) continue;
        size_t smem = (size_t)(pl->inc_words + w * pl->cand_words) * 4;
        if (smem <= (size_t)I->max_smem_optin) {
            pl->warps = w;
            pl->gstate = false;
            pl->cfg.smem = smem;
            break;
        }
    }
    // A candidate so large that shared memory holds at most 2 per SM (config 5: 32 x 256) runs
    // faster from L2-resident global scratch (per-warp state 70 KB, mostly L1/L2 hits) with 16 warps
    // per SM: one 16-warp block sharing one copy of the incumbent, 122 registers (PS_MIN_BLOCKS_G).
    if (!pl->gstate && (size_t)(pl->inc_words + pl->warps * pl->cand_words) * 4 * 2 > (size_t)I->max_smem_optin &&
        pl->warps <= 2 && env_int("PS_FORCE_SMEM", 0) == 0)
        pl->gstate = true;
    // resident blocks per SM of a plan (cached occupancy answers: one query per shape)
    auto blocks_per_sm = [&](int *per_sm) -> int {
        Variant v;
        v.gstate = pl->gstate;
        v.record = false;
        v.derived = true;
        v.uni = I->uniform != 0;
        v.wmask = pl->gstate && wmask_shape(I->MW);
        v.nobase = nobase_build(moves, pl->gstate, false, has_base, pl->cand_words);
        const uint64_t okey = ((uint64_t)pl->cfg.smem << 16) | ((uint64_t)pl->cfg.block << 3) |
                              ((uint64_t)v.nobase << 2) | ((uint64_t)pl->gstate << 1) | (uint64_t)moves;
        *per_sm = 0;
        {
            std::lock_guard<std::mutex> lk(I->occ_mu);
            auto it = I->occ_cache.find(okey);
            if (it != I->occ_cache.end()) *per_sm = it->second;
        }
        if (*per_sm == 0) {
            cudaError_t e = occupancy(I->v64, moves, v, pl->cfg.block, pl->cfg.smem, per_sm);
            if (e != cudaSuccess) return cuda_fail(e, "occupancy");
            std::lock_guard<std::mutex> lk(I->occ_mu);
            I->occ_cache[okey] = *per_sm > 0 ? *per_sm : 1;
        }
        if (*per_sm < 1) *per_sm = 1;
        return PS_OK;
    };
    auto use_gstate = [&]() {
        // global-memory state. Move mode: the warps of a block share one shared-memory copy of
        // the incumbent (48 KB at config 5), so 1-warp blocks left only 4 warps per SM resident.
        pl->gstate = true;
        pl->warps = moves ? std::max(1, std::min(PS_GSTATE_MAX_WARPS, env_int("PS_GSTATE_WARPS", PS_GSTATE_MAX_WARPS))) : 1;
        // behind it, each warp's offload / pending-transfer bitsets (read on most events); fewer
        // warps per block when a large incumbent leaves no room for all of theirs (P = 32, m = 1024)
        const int bits_w = (3 * I->P * I->MW + 3) & ~3;
        while (pl->warps > 1 && (size_t)(pl->inc_words + pl->warps * bits_w) * 4 > (size_t)I->max_smem_optin)
            pl->warps = (pl->warps + 1) / 2;
        pl->cfg.smem = (size_t)(pl->inc_words + pl->warps * bits_w) * 4;
        // and, when they fit, their ledger windows (the event loop's other hot words)
        const size_t win = (size_t)pl->warps * I->P * 2 * pl->K * ((I->v64 ? 2 : 1) + 1) * 4;
        pl->win_smem = env_int("PS_WIN_SMEM", 1) != 0 &&
                       pl->cfg.smem + win <= (size_t)env_int("PS_WIN_SMEM_MAX", I->max_smem_optin);
        if (pl->win_smem) pl->cfg.smem += win;
        pl->cfg.block = 32 * pl->warps;
    };
    int per_sm = 0, rc;
    if (pl->gstate) {
        use_gstate();
    } else {
        pl->cfg.block = 32 * pl->warps;
        if ((rc = blocks_per_sm(&per_sm)) != PS_OK) return rc;
        // Shared-memory state that leaves fewer than PS_GSTATE_BELOW_WARPS warps resident per SM
        // loses to L1/L2-resident global scratch at 16 warps (config 4, 16 x 128: 2 blocks of 4
        // warps per SM, 7.96 vs 5.61 ms per 65,536-neighbour round; configs 2 and 3 keep 28 warps
        // in shared memory, where global state is 30-50% slower; r01 tools/ab_force_g.sh). The
        // materialised config-4 kernel fits one 4-warp block per SM: e2e 25.4 -> 16.5 ms per step.
        if (env_int("PS_GSTATE_RULE", 1) && env_int("PS_FORCE_SMEM", 0) == 0 &&
            per_sm * pl->warps < env_int("PS_GSTATE_BELOW_WARPS", 12))
            use_gstate();
    }
    if (pl->cfg.smem > (size_t)I->max_smem_optin)
        return fail(PS_ERR_RANGE, "incumbent does not fit in shared memory");
    if (pl->gstate && (rc = blocks_per_sm(&per_sm)) != PS_OK) return rc;
    int64_t want = (N + pl->warps - 1) / pl->warps;
    // global state: at most 16 blocks per SM, except the no-base build's one-warp blocks
    const bool gnb = pl->gstate && nobase_build(moves, true, false, has_base, pl->cand_words);
    int64_t cap = pl->gstate && !gnb ? std::min<int64_t>(per_sm, env_int("PS_GSTATE_BLOCKS_PER_SM", 16)) * I->num_sms
                                     : (int64_t)per_sm * I->num_sms;
    pl->cfg.grid = (int)std::max<int64_t>(1, std::min<int64_t>(want, cap));
    pl->scratch_bytes = pl->gstate ? (size_t)pl->cfg.grid * pl->warps * pl->cand_words * 4 : 0;
    return PS_OK;
}

void fill_instance(const ps_instance *I, EvalParams *p) {
    p->P = I->P; p->m = I->m; p->G = I->G; p->L = I->L; p->MW = I->MW; p->stride = I->stride;
    p->comm = I->comm; p->toff = I->toff; p->post = I->post; p->uniform = I->uniform;
    p->any_off = I->any_off; p->busy = I->busy; p->unit = I->unit; p->time_safe = I->time_safe;
    p->proc = I->d_proc; p->vals = I->d_vals; p->limit = I->d_limit; p->chan = I->d_chan;
}

void attach_base(const ps_base *B, EvalParams *p) {
    p->ck = B->ck;
    p->cstep = B->cstep;
    p->fstep = B->fstep;
    p->base_info = B->info;
    p->base_res = B->res;
    p->base_orders = B->orders;
    p->base_mask = B->mask;
    p->base_chorders = B->chorders;
    p->chstep = B->chstep;
    p->ck_interval = B->ck_interval;
    p->ck_words = B->ck_words;
    p->ck_kc = B->K;
    p->ck_max = B->ck_max;
}

// Evaluation cascade on one stream, all scratch stream-ordered: a pass with the default window
// K1, then a shared-memory pass with a 4x wider window over the candidates whose ledger did not
// fit, then a pass with the whole 5m-point ledger (cannot overflow) over what is left.  Every pass
// reads its worklist from device memory: no host round trip.
int order_by_divergence(const ps_instance *I, const EvalParams &p, int32_t *order, cudaStream_t s);

// Pick up the last recording's info (its copy was queued behind the recording; by the time a
// round needs it, it has long landed).
void refresh_info(const ps_base *B) {
    if (!B->info_pending) return;
    // Not landed yet (the recording is still running): keep the last known values instead of
    // stalling the host — they only size the first pass's ledger window and hint whether a
    // re-recording may resume; the kernels read the recording's own info from device memory, and
    // a window that turns out too small is caught by the overflow passes, so results never
    // depend on it.
    if (env_int("PS_INFO_WAIT", 0) != 0) cudaEventSynchronize(B->info_ev);
    else if (cudaEventQuery(B->info_ev) != cudaSuccess) return;
    B->max_window = B->h_info[0] > 0 ? B->h_info[4] : -1;
    B->info_pending = false;
}

// first_list (optional, device [count][indices]): the candidates the first pass evaluates.
int run_eval(const ps_instance *I, EvalParams p, bool moves, cudaStream_t s, const ps_base *B = nullptr,
             const int32_t *first_list = nullptr) {
    if (p.N <= 0) return PS_OK;
    if (p.N > INT32_MAX) return fail(PS_ERR_RANGE, "at most 2^31-1 candidates per call");
    const int full = 5 * I->m;
    int K1 = window_size(I);
    // with a recorded base, neighbours need about the base's window: size the first pass from it
    if (B) refresh_info(B);
    if (B && B->inst == I && B->max_window >= 0 && !getenv("PS_WINDOW"))
        K1 = std::min(full, std::max(8, B->max_window + 4));
    int Ks[3] = {K1, std::min(full, 4 * K1), full};
    int npass = 1;
    if (Ks[0] < full) npass = Ks[1] < full ? 3 : 2;
    // a base recorded in the batch's channel mode (explicit: with the same channel-order width)
    if (B && B->inst == I && p.tcode == nullptr &&
        (p.chorders == nullptr ? B->chan_stride == 0 : B->chan_stride > 0 && B->chan_stride == p.chan_stride))
        attach_base(B, &p);
    // worklists, one per handoff between passes: [count][N candidate indices]
    // followed by one dynamic-distribution counter per pass
    int32_t *lists = nullptr;
    const size_t list_words = (size_t)p.N + 1;
    PS_CUDA(cudaMallocAsync((void **)&lists, (2 * list_words + 4) * sizeof(int32_t), s));
    PS_CUDA(cudaMemsetAsync(lists, 0, sizeof(int32_t), s));
    PS_CUDA(cudaMemsetAsync(lists + list_words, 0, sizeof(int32_t), s));
    PS_CUDA(cudaMemsetAsync(lists + 2 * list_words, 0, 4 * sizeof(int32_t), s));
    const bool dynamic = env_int("PS_DYNAMIC", 1) != 0;
    // Neighbours that diverge from the base early simulate the most: the first pass takes them
    // first (longest-processing-time order), so the round does not end on a few long stragglers.
    int32_t *order = nullptr;
    if (moves && p.ck && dynamic && env_int("PS_ORDER", 1) != 0) {
        PS_CUDA(cudaMallocAsync((void **)&order, list_words * sizeof(int32_t), s));
        int rc = order_by_divergence(I, p, order, s);
        if (rc) return rc;
    }
    for (int k = 0; k < npass; ++k) {
        Plan pl;
        int rc = plan_pass(I, moves, Ks[k], p.N, &pl, p.order_u8 ? 1 : 2, p.ck != nullptr);
        if (rc) return rc;
        EvalParams q = p;
        q.K = pl.K;
        q.cand_words = pl.cand_words;
        q.inc_words = pl.inc_words;
        q.win_smem = pl.gstate && pl.win_smem;
        const int32_t *in = k > 0 ? lists + (size_t)(k - 1) * list_words : order ? order : first_list;   // handoff k-1
        int32_t *out = k + 1 < npass ? lists + (size_t)k * list_words : nullptr;      // handoff k
        q.work_count = in;
        q.work_list = in ? in + 1 : nullptr;
        q.ovf_count = out;
        q.ovf_list = out ? out + 1 : nullptr;
        q.work_next = dynamic ? lists + 2 * list_words + k : nullptr;
        if (k > 0) q.ready = nullptr;       // later passes start after the first has read everything
        uint32_t *scratch = nullptr;
        if (pl.scratch_bytes) PS_CUDA(cudaMallocAsync((void **)&scratch, pl.scratch_bytes, s));
        q.gstate = scratch;
        cudaError_t e = launch(I->v64, moves, pl.gstate, q, pl.cfg, s);
        if (e != cudaSuccess) return cuda_fail(e, k ? "evaluator overflow pass" : "evaluator launch");
        if (scratch) PS_CUDA(cudaFreeAsync(scratch, s));
    }
    PS_CUDA(cudaFreeAsync(lists, s));
    if (order) PS_CUDA(cudaFreeAsync(order, s));
    return PS_OK;
}

// ---- search helpers ------------------------------------------------------------------------

struct MoveCtx {
    int P, m, L, stride, mask_words, uniform, any_off;
    const void *vals;
    bool v64;
};

__device__ bool ctx_offloadable(const MoveCtx &c, int s, int j) {
    int idx = (c.uniform ? s : s * c.m + j) * 4 + 3;
    if (c.v64) return reinterpret_cast<const long long *>(c.vals)[idx] > 0;
    return reinterpret_cast<const int *>(c.vals)[idx] > 0;
}

__device__ Move ctx_decode(const MoveCtx &c, const ps_move_params &mp, uint64_t round, uint64_t index) {
    return decode_move(mp.seed, round, index, c.P, c.m, mp.shift_permille, mp.max_shift,
                       c.any_off != 0, [&](int s, int j) { return ctx_offloadable(c, s, j); });
}

// One warp per (neighbour, stage) row.
__global__ void materialize_kernel(MoveCtx c, ps_move_params mp, uint64_t round, int64_t first,
                                   int64_t count, const uint16_t *inc, const uint32_t *inc_mask,
                                   uint16_t *out, uint32_t *out_mask) {
    int64_t row = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    int lane = threadIdx.x & 31;
    if (row >= count * c.P) return;
    int64_t n = row / c.P;
    int s = (int)(row % c.P);
    Move mv = ctx_decode(c, mp, round, (uint64_t)(first + n));
    const uint16_t *src = inc + (size_t)s * c.stride;
    uint16_t *dst = out + ((size_t)n * c.P + s) * c.stride;
    bool shift = mv.type == MOVE_SHIFT && mv.stage == s;
    for (int q = lane; q < c.stride; q += 32)
        dst[q] = q < c.L ? src[shift ? shifted_position(q, mv.a, mv.b) : q] : (uint16_t)0;
    if (s == 0)
        for (int w = lane; w < c.mask_words; w += 32) {
            uint32_t v = inc_mask[w];
            if (mv.type == MOVE_TOGGLE) {
                int b = mv.stage * c.m + mv.mb;
                if ((b >> 5) == w) v ^= 1u << (b & 31);
            }
            out_mask[(size_t)n * c.mask_words + w] = v;
        }
}

__global__ void apply_move_kernel(MoveCtx c, ps_move_params mp, uint64_t round, uint64_t index,
                                  uint16_t *inc, uint32_t *inc_mask) {
    if (threadIdx.x) return;
    Move mv = ctx_decode(c, mp, round, index);
    if (mv.type == MOVE_SHIFT) {
        uint16_t *row = inc + (size_t)mv.stage * c.stride;
        uint16_t v = row[mv.a];
        if (mv.a < mv.b)
            for (int q = mv.a; q < mv.b; ++q) row[q] = row[q + 1];
        else
            for (int q = mv.a; q > mv.b; --q) row[q] = row[q - 1];
        row[mv.b] = v;
    } else if (mv.type == MOVE_TOGGLE) {
        int b = mv.stage * c.m + mv.mb;
        inc_mask[b >> 5] ^= 1u << (b & 31);
    }
}

// A re-recording that converged onto the previous base at checkpoint c0 with time shift dl
// (base info[5], info[6]): every later checkpoint is the previous base's with each live time
// moved by dl — F/B/transfer end words, ledger breakpoints, stage and used-channel free times —
// the new base's offload bits and first starts, and the new peak prefix.  One block per
// checkpoint.
struct RecShift {
    int P, m, MW, mask_words, ck_words, ck_kc, ck_t, ck_r, ck_max;
    uint32_t *ck;
    const int32_t *info;
    const uint32_t *mask;
};

__global__ void rec_shift_kernel(RecShift r) {
    const int c0 = r.info[5];
    const int c = blockIdx.x;
    if (c0 < 0 || c <= c0 || c >= r.info[0]) return;
    const int dl = r.info[6];
    uint32_t *ck = r.ck + (size_t)c * r.ck_words;
    const uint32_t d4 = (uint32_t)dl << 2;
    for (int k = threadIdx.x; k < 2 * r.P * r.m; k += blockDim.x) {
        const uint32_t w = ck[k];
        if ((w >> 2) && w != ps::A_DEAD) ck[k] = w + d4;      // words that carry a time
    }
    for (int k = threadIdx.x; k < r.P * r.MW; k += blockDim.x) {
        const int s = k / r.MW, w = k % r.MW;
        const int gb = s * r.m + w * 32, q = gb >> 5, sh = gb & 31;
        uint32_t bits = (q < r.mask_words ? r.mask[q] : 0u) >> sh;
        if (sh && q + 1 < r.mask_words) bits |= r.mask[q + 1] << (32 - sh);
        const int nb = r.m - w * 32;
        if (nb < 32) bits &= (1u << nb) - 1u;
        ck[2 * r.P * r.m + k] = bits;
    }
    // the event step is a warp-wide scalar: every lane's copy moves
    for (int l = threadIdx.x; l < 32; l += blockDim.x) ck[r.ck_r + l * ps::CK_REGW + 20] -= (uint32_t)r.info[7];
    const uint32_t *rg0 = r.ck + (size_t)c0 * r.ck_words + r.ck_r;
    for (int s = threadIdx.x; s < r.P; s += blockDim.x) {
        uint32_t *rg = ck + r.ck_r + s * ps::CK_REGW;
        const int count = (int)rg[4];
        for (int q = 0; q < count; ++q) ck[r.ck_t + s * r.ck_kc + q] += (uint32_t)dl;
        rg[1] += (uint32_t)dl;
        if (rg[2]) rg[2] += (uint32_t)dl;
        const int fs0 = (int)rg0[s * ps::CK_REGW + 8];
        if (fs0 != INT_MAX) rg[8] = (uint32_t)fs0;
        else if ((int)rg[8] != INT_MAX) rg[8] += (uint32_t)dl;
        long long pk = *reinterpret_cast<const long long *>(rg0 + s * ps::CK_REGW + 16);
        for (int k = c0 + 1; k <= c; ++k) {
            const long long sg = *reinterpret_cast<const long long *>(r.ck + (size_t)k * r.ck_words + r.ck_r + s * ps::CK_REGW + 10);
            pk = sg > pk ? sg : pk;
        }
        *reinterpret_cast<long long *>(rg + 16) = pk;
    }
}

// Divergence step of every neighbour of a round (the base's compute index before which the
// neighbour's inputs first differ; NEVER for no-ops), with its index, for the LPT ordering.
MoveCtx move_ctx(const ps_instance *I);

__global__ void divergence_kernel(MoveCtx c, ps_move_params mp, uint64_t round, int64_t first, int64_t count,
                                  const uint32_t *cstep, const uint32_t *fstep, uint32_t *key, int32_t *idx,
                                  int32_t *order_count, const unsigned long long *move_list) {
    const int64_t n = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (n == 0) *order_count = (int32_t)count;
    if (n >= count) return;
    const Move mv = move_list ? unpack_move(move_list[n]) : ctx_decode(c, mp, round, (uint64_t)(first + n));
    uint32_t d = ps::NEVER;
    if (mv.type == MOVE_SHIFT) {
        const int q = mv.a < mv.b ? mv.a : mv.b;
        d = q == 0 ? 0u : cstep[mv.stage * c.L + q - 1];
    } else if (mv.type == MOVE_TOGGLE) {
        d = fstep[mv.stage * c.m + mv.mb];
    }
    // (no-ops and never-reached steps sort last: keys stay below 3Pm + 1, so the radix sort only
    // needs the bits of 3Pm)
    const uint32_t last = (uint32_t)(c.P * c.L);
    key[n] = d < last ? d : last;
    idx[n] = (int32_t)n;
}

// Distinct moves of a round, in LPT order: key = divergence:15 | shift:1 | stage:5 | a:13 | b:13 |
// index:17 (an adjacent shift a->a+1 is the same permutation as a+1->a; a no-op has a = b = 8191).
// Dedup keys, packed as tightly as the instance allows (fewer radix passes):
// divergence (db bits, never-reached capped at 3Pm) | shift? | stage (sb) | a (ab) | b (ab) | index (17).
struct DedupLayout {
    int db, sb, ab;
};

__global__ void dedup_key_kernel(MoveCtx c, ps_move_params mp, uint64_t round, int64_t first, int64_t count,
                                 const uint32_t *cstep, const uint32_t *fstep, DedupLayout lay,
                                 unsigned long long *key) {
    const int64_t n = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (n >= count) return;
    const Move mv = ctx_decode(c, mp, round, (uint64_t)(first + n));
    const uint32_t dmax = (uint32_t)(c.P * c.L), none = (1u << lay.ab) - 1u;
    uint32_t d = dmax, sh = 0, st = 0, a = none, bb = none;
    if (mv.type == MOVE_SHIFT) {
        const int q = mv.a < mv.b ? mv.a : mv.b;
        d = q == 0 ? 0u : cstep[mv.stage * c.L + q - 1];
        sh = 1; st = mv.stage; a = mv.a; bb = mv.b;
        if (mv.a - mv.b == 1 || mv.b - mv.a == 1) { a = q; bb = q + 1; }
    } else if (mv.type == MOVE_TOGGLE) {
        d = fstep[mv.stage * c.m + mv.mb];
        st = mv.stage; a = mv.mb; bb = 0;
    }
    if (d > dmax) d = dmax;
    const int pb = 17, pa = pb + lay.ab, ps = pa + lay.ab, psh = ps + lay.sb, pd = psh + 1;
    key[n] = ((unsigned long long)d << pd) | ((unsigned long long)sh << psh) | ((unsigned long long)st << ps) |
             ((unsigned long long)a << pa) | ((unsigned long long)bb << pb) | (unsigned long long)n;
}

__global__ void dedup_head_kernel(const unsigned long long *sorted, int64_t count, int32_t *idx, unsigned char *head) {
    const int64_t n = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (n >= count) return;
    idx[n] = (int32_t)(sorted[n] & 0x1FFFFull);
    head[n] = n == 0 || (sorted[n] >> 17) != (sorted[n - 1] >> 17);
}

int order_by_divergence(const ps_instance *I, const EvalParams &p, int32_t *order, cudaStream_t s) {
    const int64_t N = p.N;
    ps_move_params mp;
    mp.seed = p.seed;
    mp.shift_permille = p.shift_permille;
    mp.max_shift = p.max_shift;
    auto bits_of = [](int64_t v) { int b = 1; while (b < 63 && (v >> b)) ++b; return b; };
    DedupLayout lay;
    lay.db = bits_of((int64_t)I->P * I->L);
    lay.sb = bits_of(I->P - 1);
    lay.ab = bits_of(I->L);
    const int key_bits64 = lay.db + 1 + lay.sb + 2 * lay.ab + 17;
    if (p.dedup && N <= (1 << 17) && key_bits64 <= 64) {
        // the same move drawn several times in a round is simulated once: its lowest index
        // carries it, so the round's best key is unchanged
        unsigned long long *keys = nullptr, *sorted = nullptr;
        int32_t *idx = nullptr;
        unsigned char *head = nullptr;
        void *tmp = nullptr;
        size_t b1 = 0, b2 = 0;
        PS_CUDA(cub::DeviceRadixSort::SortKeys(nullptr, b1, keys, sorted, (int)N, 0, key_bits64, s));
        PS_CUDA(cub::DeviceSelect::Flagged(nullptr, b2, idx, head, order + 1, order, (int)N, s));
        PS_CUDA(cudaMallocAsync((void **)&keys, (size_t)N * 8, s));
        PS_CUDA(cudaMallocAsync((void **)&sorted, (size_t)N * 8, s));
        PS_CUDA(cudaMallocAsync((void **)&idx, (size_t)N * 4, s));
        PS_CUDA(cudaMallocAsync((void **)&head, (size_t)N, s));
        PS_CUDA(cudaMallocAsync(&tmp, std::max(b1, b2), s));
        const unsigned g = (unsigned)((N + 255) / 256);
        dedup_key_kernel<<<g, 256, 0, s>>>(move_ctx(I), mp, p.round, p.first_index, N, p.cstep, p.fstep, lay, keys);
        PS_CUDA(cudaGetLastError());
        size_t tb = std::max(b1, b2);
        PS_CUDA(cub::DeviceRadixSort::SortKeys(tmp, tb, keys, sorted, (int)N, 0, key_bits64, s));
        dedup_head_kernel<<<g, 256, 0, s>>>(sorted, N, idx, head);
        PS_CUDA(cudaGetLastError());
        tb = std::max(b1, b2);
        PS_CUDA(cub::DeviceSelect::Flagged(tmp, tb, idx, head, order + 1, order, (int)N, s));
        cudaFreeAsync(keys, s);
        cudaFreeAsync(sorted, s);
        cudaFreeAsync(idx, s);
        cudaFreeAsync(head, s);
        cudaFreeAsync(tmp, s);
        return PS_OK;
    }
    uint32_t *keys = nullptr, *keys_out = nullptr;
    int32_t *idx = nullptr;
    void *tmp = nullptr;
    size_t tmp_bytes = 0;
    int key_bits = 1;
    while (key_bits < 32 && ((int64_t)I->P * I->L) >> key_bits) ++key_bits;
    PS_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tmp_bytes, keys, keys_out, idx, order + 1, (int)N, 0, key_bits, s));
    PS_CUDA(cudaMallocAsync((void **)&keys, (size_t)N * 4, s));
    PS_CUDA(cudaMallocAsync((void **)&keys_out, (size_t)N * 4, s));
    PS_CUDA(cudaMallocAsync((void **)&idx, (size_t)N * 4, s));
    PS_CUDA(cudaMallocAsync(&tmp, tmp_bytes, s));
    divergence_kernel<<<(unsigned)((N + 255) / 256), 256, 0, s>>>(move_ctx(I), mp, p.round, p.first_index, N,
                                                                 p.cstep, p.fstep, keys, idx, order, p.move_list);
    PS_CUDA(cudaGetLastError());
    PS_CUDA(cub::DeviceRadixSort::SortPairs(tmp, tmp_bytes, keys, keys_out, idx, order + 1, (int)N, 0, key_bits, s));
    cudaFreeAsync(keys, s);
    cudaFreeAsync(keys_out, s);
    cudaFreeAsync(idx, s);
    cudaFreeAsync(tmp, s);
    return PS_OK;
}

// Independent IADD3/LOP3/IMAD chains: the INT32 issue ceiling of the roofline.
__global__ void int32_probe_kernel(int64_t iters, uint32_t seed, unsigned long long *lane_ops, uint32_t *sink) {
    uint32_t a0 = threadIdx.x ^ seed, a1 = a0 * 3u, a2 = a0 + 7u, a3 = a0 ^ 0x55u;
    uint32_t b0 = a0 + 1u, b1 = a1 + 2u, b2 = a2 + 3u, b3 = a3 + 4u;
    for (int64_t it = 0; it < iters; ++it) {
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            a0 = (a0 + b1) ^ b2; a1 = (a1 + b2) ^ b3; a2 = (a2 + b3) ^ b0; a3 = (a3 + b0) ^ b1;
            b0 = b0 * 0x9E37u + a1; b1 = b1 * 0x85EBu + a2; b2 = b2 * 0xC2B2u + a3; b3 = b3 * 0x27D4u + a0;
        }
    }
    uint32_t r = a0 ^ a1 ^ a2 ^ a3 ^ b0 ^ b1 ^ b2 ^ b3;
    if (r == seed) sink[0] = r;   // keeps the chains alive
    if (threadIdx.x == 0 && blockIdx.x == 0)
        atomicAdd(lane_ops, (unsigned long long)iters * 8ull * 12ull * blockDim.x * gridDim.x);
}

MoveCtx move_ctx(const ps_instance *I) {
    MoveCtx c;
    c.P = I->P; c.m = I->m; c.L = I->L; c.stride = I->stride; c.mask_words = I->mask_words;
    c.uniform = I->uniform; c.any_off = I->any_off; c.vals = I->d_vals; c.v64 = I->v64;
    return c;
}

}  // namespace

// =============================================================================================
extern "C" {

const char *ps_version(void) { return "pipesched_b200 0.1.0 (sm_100a)"; }

const char *ps_last_error(void) { return g_last_error.c_str(); }

int ps_instance_create(const ps_instance_desc *d, int device, ps_instance **out) {
    if (!d || !out) return fail(PS_ERR_INVALID, "null argument");
    *out = nullptr;
    const int P = d->num_stages, m = d->num_microbatches;
    if (P < 1 || P > PS_MAX_STAGES) return fail(PS_ERR_RANGE, "num_stages %d outside 1..%d", P, PS_MAX_STAGES);
    if (m < 1 || m > PS_MAX_MICROBATCHES)
        return fail(PS_ERR_RANGE, "num_microbatches %d outside 1..%d", m, PS_MAX_MICROBATCHES);
    if (!d->proc_time || !d->mem_delta || !d->act_size || !d->mem_limit || !d->stage_channel)
        return fail(PS_ERR_INVALID, "null table");
    if (d->comm_time < 0 || d->offload_time < 0) return fail(PS_ERR_INVALID, "comm_time and offload_time must be >= 0");
    if (d->num_channels < 1 || d->num_channels > P) return fail(PS_ERR_INVALID, "num_channels %d", d->num_channels);
    // instance invariants (reference instance.py:88-126)
    int64_t unit = 0, busy = 0, n_off = 0;
    bool uniform = true, any_off = false;
    for (int i = 0; i < P; ++i) {
        if (d->mem_limit[i] <= 0) return fail(PS_ERR_INVALID, "mem_limit must be positive for stage %d", i + 1);
        if (d->stage_channel[i] < 0 || d->stage_channel[i] >= d->num_channels)
            return fail(PS_ERR_INVALID, "stage %d has channel %d", i + 1, d->stage_channel[i]);
        unit = gcd64(unit, d->mem_limit[i]);
        for (int j = 0; j < m; ++j) {
            const int64_t *t = d->proc_time + ((size_t)i * m + j) * 3;
            const int64_t *v = d->mem_delta + ((size_t)i * m + j) * 3;
            int64_t g = d->act_size[(size_t)i * m + j];
            for (int k = 0; k < 3; ++k) {
                if (t[k] <= 0) return fail(PS_ERR_INVALID, "proc_time must be positive at (%d,%d,%d)", i + 1, j + 1, k);
                busy += t[k];
                unit = gcd64(unit, v[k]);
            }
            if (v[0] + v[1] + v[2] != 0) return fail(PS_ERR_INVALID, "mem_delta sum nonzero for stage %d microbatch %d", i + 1, j + 1);
            if (!(v[0] > 0 && v[1] < 0 && v[2] < 0))
                return fail(PS_ERR_INVALID, "mem_delta signs wrong for stage %d microbatch %d", i + 1, j + 1);
            if (g < 0 || g > v[0]) return fail(PS_ERR_INVALID, "act_size outside [0, mem_delta_F] at stage %d microbatch %d", i + 1, j + 1);
            if (g > 0) { unit = gcd64(unit, g); any_off = true; ++n_off; }
            if (j > 0) {
                const int64_t *t0 = d->proc_time + (size_t)i * m * 3;
                const int64_t *v0 = d->mem_delta + (size_t)i * m * 3;
                for (int k = 0; k < 3; ++k)
                    if (t[k] != t0[k] || v[k] != v0[k]) uniform = false;
                if (g != d->act_size[(size_t)i * m]) uniform = false;
            }
        }
    }
    // Event times are packed as (t << 2 | state) in 32 bits, so every event must end below 2^29.
    // Durations must fit well inside that; the instance's horizon (no event of any structure can
    // end later) decides whether the kernels check at all: past it, an event chosen to start at or
    // after 2^29 - (longest duration) ends that candidate with PS_FLAG_RANGE (ps_eval.cuh), and
    // ps_eval_batch finishes it in 64-bit time (ps_literal.cu): instances with long horizons are
    // accepted and every candidate is exact.  (Search rounds do not adopt such a neighbour.)
    int64_t max_dur = std::max<int64_t>(d->comm_time, d->offload_time);
    for (size_t k = 0; k < (size_t)P * m * 3; ++k) max_dur = std::max<int64_t>(max_dur, d->proc_time[k]);
    if (max_dur >= (int64_t)1 << 27)
        return fail(PS_ERR_RANGE, "a duration of %lld quanta exceeds the 2^27 range", (long long)max_dur);
    double horizon = (double)busy + 2.0 * n_off * d->offload_time + (2.0 * m * P + 1.0) * d->comm_time;
    const int time_safe = horizon < (double)(1 << 29) ? INT_MAX : (int)((1 << 29) - max_dur);
    // ledger width: usage never exceeds the sum of a stage's F deltas
    bool v64 = false;
    for (int i = 0; i < P; ++i) {
        int64_t s = d->mem_limit[i] / unit;
        for (int j = 0; j < m; ++j) s += d->mem_delta[((size_t)i * m + j) * 3] / unit;
        if (s > (int64_t)(INT32_MAX / 4)) v64 = true;
    }

    ps_instance *I = new (std::nothrow) ps_instance();
    if (!I) return fail(PS_ERR_NOMEM, "host allocation");
    I->device = device;
    I->P = P; I->m = m; I->G = d->num_channels; I->L = 3 * m; I->MW = (m + 31) / 32;
    I->stride = (3 * m + 7) & ~7;
    I->mask_words = (P * m + 31) / 32;
    I->comm = (int)d->comm_time; I->toff = (int)d->offload_time; I->post = d->post_validation != 0;
    I->uniform = uniform; I->any_off = any_off; I->busy = busy; I->unit = unit; I->v64 = v64;
    I->time_safe = time_safe;
    I->h_offloadable.resize((size_t)P * m);
    for (size_t k = 0; k < (size_t)P * m; ++k) I->h_offloadable[k] = d->act_size[k] > 0;

    DeviceGuard guard(device);
    if (!guard.ok) { delete I; return fail(PS_ERR_CUDA, "cannot select device %d", device); }
    cudaDeviceProp prop;
    cudaError_t e = cudaGetDeviceProperties(&prop, device);
    if (e != cudaSuccess) { delete I; return cuda_fail(e, "cudaGetDeviceProperties"); }
    I->num_sms = prop.multiProcessorCount;
    I->max_smem_optin = (int)prop.sharedMemPerBlockOptin;
    {
        cudaMemPool_t pool;
        if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) {
            uint64_t thr = UINT64_MAX;
            cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
        }
    }

    const int rows = uniform ? P : P * m;
    std::vector<int32_t> proc((size_t)rows * 3), chan(P);
    std::vector<int64_t> vals64((size_t)rows * 4), lim64(P);
    for (int r = 0; r < rows; ++r) {
        size_t src = uniform ? (size_t)r * m : (size_t)r;   // uniform: row r = stage r, microbatch 0
        for (int k = 0; k < 3; ++k) {
            proc[(size_t)r * 3 + k] = (int32_t)d->proc_time[src * 3 + k];
            vals64[(size_t)r * 4 + k] = d->mem_delta[src * 3 + k] / unit;
        }
        vals64[(size_t)r * 4 + 3] = d->act_size[src] / unit;
    }
    for (int i = 0; i < P; ++i) {
        lim64[i] = d->mem_limit[i] / unit;
        chan[i] = d->stage_channel[i];
    }
    size_t vb = v64 ? 8 : 4;
    e = cudaMalloc((void **)&I->d_proc, proc.size() * 4);
    if (e == cudaSuccess) e = cudaMalloc(&I->d_vals, vals64.size() * vb);
    if (e == cudaSuccess) e = cudaMalloc(&I->d_limit, (size_t)P * vb);
    if (e == cudaSuccess) e = cudaMalloc((void **)&I->d_chan, (size_t)P * 4);
    if (e != cudaSuccess) { ps_instance_destroy(I); return fail(PS_ERR_NOMEM, "device tables: %s", cudaGetErrorString(e)); }
    std::vector<int32_t> vals32, lim32;
    const void *vsrc = vals64.data(), *lsrc = lim64.data();
    if (!v64) {
        vals32.assign(vals64.begin(), vals64.end());
        lim32.assign(lim64.begin(), lim64.end());
        vsrc = vals32.data();
        lsrc = lim32.data();
    }
    e = cudaMemcpy(I->d_proc, proc.data(), proc.size() * 4, cudaMemcpyHostToDevice);
    if (e == cudaSuccess) e = cudaMemcpy(I->d_vals, vsrc, vals64.size() * vb, cudaMemcpyHostToDevice);
    if (e == cudaSuccess) e = cudaMemcpy(I->d_limit, lsrc, (size_t)P * vb, cudaMemcpyHostToDevice);
    if (e == cudaSuccess) e = cudaMemcpy(I->d_chan, chan.data(), (size_t)P * 4, cudaMemcpyHostToDevice);
    if (e != cudaSuccess) { ps_instance_destroy(I); return cuda_fail(e, "upload instance tables"); }
    *out = I;
    return PS_OK;
}

int ps_instance_destroy(ps_instance *I) {
    if (!I) return PS_OK;
    DeviceGuard guard(I->device);
    cudaFree(I->d_proc);
    cudaFree(I->d_vals);
    cudaFree(I->d_limit);
    cudaFree(I->d_chan);
    delete I;
    return PS_OK;
}

int ps_instance_get_info(const ps_instance *I, ps_instance_info *o) {
    if (!I || !o) return fail(PS_ERR_INVALID, "null argument");
    o->num_stages = I->P;
    o->num_microbatches = I->m;
    o->order_stride = I->stride;
    o->mask_words = I->mask_words;
    o->max_events = 5 * I->P * I->m;
    o->value_bits = I->v64 ? 64 : 32;
    o->memory_unit = I->unit;
    o->busy_time = I->busy;
    o->lanes_per_candidate = 32;
    o->device = I->device;
    return PS_OK;
}

int ps_base_create(const ps_instance *I, ps_base **out) {
    if (!I || !out) return fail(PS_ERR_INVALID, "null argument");
    *out = nullptr;
    DeviceGuard guard(I->device);
    if (!guard.ok) return fail(PS_ERR_CUDA, "cannot select device %d", I->device);
    ps_base *B = new (std::nothrow) ps_base();
    if (!B) return fail(PS_ERR_NOMEM, "host allocation");
    B->inst = I;
    B->K = (std::min(5 * I->m, 128) + 1) & ~1;     // recording window (checkpoints store it compactly);
                                                    // even, like a pass's (16-byte aligned state words)
    B->max_window = -1;
    B->cand_words = words_per_candidate(I, B->K, 2);
    {
        const int vw = I->v64 ? 2 : 1;
        const int nz = 2 * I->P * I->m + 3 * I->P * I->MW;
        const int ck_t = (nz + 1) & ~1;
        const int ck_u = (ck_t + I->P * B->K + 1) & ~1;
        B->ck_words = (ck_u + I->P * B->K * vw + 32 * CK_REGW + 3) & ~3;   // 16-byte aligned checkpoints
    }
    // checkpoints every ck_interval compute events (3Pm per candidate)
    B->ck_interval = std::max(1, next_pow2(std::max(1, env_int("PS_CHECKPOINT_INTERVAL", 8))));
    B->ck_max = 3 * I->P * I->m / B->ck_interval + 2;
    cudaError_t e = cudaMalloc((void **)&B->ck, (size_t)B->ck_max * B->ck_words * 4);
    if (e == cudaSuccess) e = cudaMalloc((void **)&B->cstep, (size_t)I->P * I->L * 4);
    if (e == cudaSuccess) e = cudaMalloc((void **)&B->fstep, (size_t)I->P * I->m * 4);
    if (e == cudaSuccess) e = cudaMalloc((void **)&B->info, 8 * sizeof(int32_t));
    if (e == cudaSuccess) e = cudaMalloc((void **)&B->res, (size_t)(2 + 3 * I->P) * sizeof(int64_t));
    if (e == cudaSuccess) e = cudaMalloc((void **)&B->orders, (size_t)I->P * I->stride * 2);
    if (e == cudaSuccess) e = cudaMalloc((void **)&B->mask, (size_t)I->mask_words * 4);
    if (e == cudaSuccess) e = cudaMalloc((void **)&B->prev_orders, (size_t)I->P * I->stride * 2);
    if (e == cudaSuccess) e = cudaMalloc((void **)&B->prev_mask, (size_t)I->mask_words * 4);
    if (e == cudaSuccess) e = cudaMemset(B->info, 0xFF, 8 * sizeof(int32_t));   // -1: nothing recorded
    if (e == cudaSuccess) e = cudaHostAlloc((void **)&B->h_info, 8 * sizeof(int32_t), cudaHostAllocDefault);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&B->info_ev, cudaEventDisableTiming);
    if (e != cudaSuccess) {
        ps_base_destroy(B);
        return fail(PS_ERR_NOMEM, "base workspace: %s", cudaGetErrorString(e));
    }
    *out = B;
    return PS_OK;
}

int ps_base_destroy(ps_base *B) {
    if (!B) return PS_OK;
    DeviceGuard guard(B->inst->device);
    cudaFree(B->ck);
    cudaFree(B->cstep);
    cudaFree(B->fstep);
    cudaFree(B->info);
    cudaFree(B->res);
    cudaFree(B->orders);
    cudaFree(B->mask);
    cudaFree(B->prev_orders);
    cudaFree(B->prev_mask);
    cudaFree(B->chorders);
    cudaFree(B->prev_chorders);
    cudaFree(B->chstep);
    if (B->info_pending) cudaEventSynchronize(B->info_ev);
    if (B->h_info) cudaFreeHost(B->h_info);
    if (B->info_ev) cudaEventDestroy(B->info_ev);
    delete B;
    return PS_OK;
}

static int check_x(const ps_instance *I, const uint32_t *inc_chan, int chan_stride);

static int base_record_impl(ps_base *B, const uint16_t *orders, const uint32_t *mask, const uint32_t *chan,
                            int32_t chan_stride, void *stream) {
    NvtxRange nvtx("ps_base_record");
    if (!B || !orders || !mask) return fail(PS_ERR_INVALID, "null argument");
    const ps_instance *I = B->inst;
    DeviceGuard guard(I->device);
    if (!guard.ok) return fail(PS_ERR_CUDA, "cannot select device %d", I->device);
    cudaStream_t s = (cudaStream_t)stream;
    // A usable previous recording is kept: the new base replays it up to their first difference
    // (its checkpoints, cstep and fstep entries before that point are the new base's too).
    refresh_info(B);
    const bool resume = B->max_window >= 0 && B->rec_stride == chan_stride && env_int("PS_REC_RESUME", 1) != 0;
    if (chan_stride > 0 && B->cap_stride < chan_stride) {
        // channel-order tables sized for this width (kept across recordings of the same width)
        PS_CUDA(cudaStreamSynchronize(s));
        cudaFree(B->chorders);
        cudaFree(B->prev_chorders);
        cudaFree(B->chstep);
        B->chorders = B->prev_chorders = B->chstep = nullptr;
        B->cap_stride = 0;
        const size_t nb = (size_t)I->G * chan_stride * 4;
        cudaError_t e = cudaMalloc((void **)&B->chorders, nb);
        if (e == cudaSuccess) e = cudaMalloc((void **)&B->prev_chorders, nb);
        if (e == cudaSuccess) e = cudaMalloc((void **)&B->chstep, nb);
        if (e != cudaSuccess) return fail(PS_ERR_NOMEM, "base channel tables: %s", cudaGetErrorString(e));
        B->cap_stride = chan_stride;
    }
    if (resume && chan_stride > 0)
        PS_CUDA(cudaMemcpyAsync(B->prev_chorders, B->chorders, (size_t)I->G * chan_stride * 4, cudaMemcpyDeviceToDevice, s));
    if (chan_stride > 0)
        PS_CUDA(cudaMemcpyAsync(B->chorders, chan, (size_t)I->G * chan_stride * 4, cudaMemcpyDeviceToDevice, s));
    B->chan_stride = chan_stride;
    B->rec_stride = chan_stride;
    if (resume) {
        PS_CUDA(cudaMemcpyAsync(B->prev_orders, B->orders, (size_t)I->P * I->stride * 2, cudaMemcpyDeviceToDevice, s));
        PS_CUDA(cudaMemcpyAsync(B->prev_mask, B->mask, (size_t)I->mask_words * 4, cudaMemcpyDeviceToDevice, s));
    }
    PS_CUDA(cudaMemcpyAsync(B->orders, orders, (size_t)I->P * I->stride * 2, cudaMemcpyDeviceToDevice, s));
    PS_CUDA(cudaMemcpyAsync(B->mask, mask, (size_t)I->mask_words * 4, cudaMemcpyDeviceToDevice, s));
    if (!resume) {
        PS_CUDA(cudaMemsetAsync(B->cstep, 0xFF, (size_t)I->P * I->L * 4, s));
        PS_CUDA(cudaMemsetAsync(B->fstep, 0xFF, (size_t)I->P * I->m * 4, s));
        if (chan_stride > 0) PS_CUDA(cudaMemsetAsync(B->chstep, 0xFF, (size_t)I->G * chan_stride * 4, s));
    }
    EvalParams p;
    memset(&p, 0, sizeof p);
    fill_instance(I, &p);
    p.N = 1;
    p.orders = B->orders;
    p.masks = B->mask;
    p.K = B->K;
    p.cand_words = B->cand_words;
    p.inc_words = 0;
    attach_base(B, &p);
    if (chan_stride > 0) {
        p.chorders = B->chorders;
        p.chan_stride = chan_stride;
    }
    if (resume) {
        p.base_orders = B->prev_orders;
        p.base_mask = B->prev_mask;
        p.base_chorders = B->prev_chorders;
        p.rec_prev = 1;
    }
    LaunchCfg cfg;
    cfg.grid = 1;
    cfg.block = 32;
    cfg.smem = (size_t)B->cand_words * 4;
    if (cfg.smem > (size_t)I->max_smem_optin) {
        // too large to record in shared memory: leave the base unusable (evaluations run in full)
        PS_CUDA(cudaMemsetAsync(B->info, 0xFF, 4 * sizeof(int32_t), s));
        return PS_OK;
    }
    cudaError_t e = launch(I->v64, false, false, p, cfg, s, true);
    if (e != cudaSuccess) return cuda_fail(e, "base recording launch");
    if (resume) {
        RecShift r;
        r.P = I->P; r.m = I->m; r.MW = I->MW; r.mask_words = I->mask_words;
        r.ck_words = B->ck_words; r.ck_kc = B->K; r.ck_max = B->ck_max;
        const int nz = 2 * I->P * I->m + 3 * I->P * I->MW;
        r.ck_t = (nz + 1) & ~1;
        const int ck_u = (r.ck_t + I->P * B->K + 1) & ~1;
        r.ck_r = ck_u + I->P * B->K * (I->v64 ? 2 : 1);
        r.ck = B->ck; r.info = B->info; r.mask = B->mask;
        rec_shift_kernel<<<B->ck_max, 128, 0, s>>>(r);
        PS_CUDA(cudaGetLastError());
    }
    // the evaluation passes size their ledger window from the base's (one host read per record)
    PS_CUDA(cudaMemcpyAsync(B->h_info, B->info, 8 * sizeof(int32_t), cudaMemcpyDeviceToHost, s));
    PS_CUDA(cudaEventRecord(B->info_ev, s));
    B->info_pending = true;
    return PS_OK;
}

int ps_base_record(ps_base *B, const uint16_t *orders, const uint32_t *mask, void *stream) {
    return base_record_impl(B, orders, mask, nullptr, 0, stream);
}

int ps_base_record_explicit(ps_base *B, const uint16_t *orders, const uint32_t *mask, const uint32_t *chan_orders,
                            int32_t chan_stride, void *stream) {
    if (!B || !chan_orders || chan_stride < 1) return fail(PS_ERR_INVALID, "channel orders and a positive width are required");
    int rc = check_x(B->inst, chan_orders, chan_stride);
    if (rc) return rc;
    return base_record_impl(B, orders, mask, chan_orders, chan_stride, stream);
}

int ps_base_read(const ps_base *B, int what, void *host, size_t *bytes) {
    if (!B || !bytes) return fail(PS_ERR_INVALID, "null argument");
    const ps_instance *I = B->inst;
    const void *src = nullptr;
    size_t n = 0;
    switch (what) {
        case PS_BASE_CHECKPOINTS: src = B->ck; n = (size_t)B->ck_max * B->ck_words * 4; break;
        case PS_BASE_CSTEP: src = B->cstep; n = (size_t)I->P * I->L * 4; break;
        case PS_BASE_FSTEP: src = B->fstep; n = (size_t)I->P * I->m * 4; break;
        case PS_BASE_INFO: src = B->info; n = 8 * sizeof(int32_t); break;
        case PS_BASE_RESULT: src = B->res; n = (size_t)(2 + 3 * I->P) * sizeof(int64_t); break;
        case PS_BASE_LAYOUT: {
            const int nz = 2 * I->P * I->m + 3 * I->P * I->MW;
            const int ck_t = (nz + 1) & ~1;
            const int ck_u = (ck_t + I->P * B->K + 1) & ~1;
            const int32_t lay[8] = {B->ck_words, B->ck_max, B->ck_interval, B->K, ck_t, ck_u,
                                    ck_u + I->P * B->K * (I->v64 ? 2 : 1), CK_REGW};
            if (!host) { *bytes = sizeof lay; return PS_OK; }
            if (*bytes < sizeof lay) return fail(PS_ERR_RANGE, "buffer too small");
            memcpy(host, lay, sizeof lay);
            *bytes = sizeof lay;
            return PS_OK;
        }
        default: return fail(PS_ERR_INVALID, "unknown base table %d", what);
    }
    if (!host) { *bytes = n; return PS_OK; }
    if (*bytes < n) return fail(PS_ERR_RANGE, "buffer of %zu bytes < %zu", *bytes, n);
    *bytes = n;
    DeviceGuard guard(I->device);
    if (!guard.ok) return fail(PS_ERR_CUDA, "cannot select device %d", I->device);
    PS_CUDA(cudaDeviceSynchronize());
    PS_CUDA(cudaMemcpy(host, src, n, cudaMemcpyDeviceToHost));
    return PS_OK;
}

static int eval_batch_impl(const ps_instance *I, const ps_cand_batch *b, const ps_result_batch *r,
                           cudaStream_t stream, const int32_t *ready, int64_t ready_chunk,
                           const int32_t *first_list = nullptr);

int ps_eval_batch(const ps_instance *I, const ps_cand_batch *b, const ps_result_batch *r, void *stream) {
    NvtxRange nvtx("ps_eval_batch n=%llu", (unsigned long long)(b ? b->num_candidates : 0));
    return eval_batch_impl(I, b, r, (cudaStream_t)stream, nullptr, 0);
}

static int eval_batch_impl(const ps_instance *I, const ps_cand_batch *b, const ps_result_batch *r,
                           cudaStream_t stream, const int32_t *ready, int64_t ready_chunk,
                           const int32_t *first_list) {
    if (!I || !b || !r) return fail(PS_ERR_INVALID, "null argument");
    if (b->num_candidates < 0) return fail(PS_ERR_INVALID, "negative candidate count");
    if (b->num_candidates == 0) return PS_OK;
    if (!b->stage_orders || !b->offload_mask) return fail(PS_ERR_INVALID, "stage_orders and offload_mask are required");
    if (!r->makespan || !r->flags || !r->bubble) return fail(PS_ERR_INVALID, "makespan, bubble and flags outputs are required");
    if (b->channel_orders && b->chan_stride < 1) return fail(PS_ERR_INVALID, "chan_stride must be positive");
    if (b->order_bytes != 0 && b->order_bytes != 1 && b->order_bytes != 2)
        return fail(PS_ERR_INVALID, "order_bytes must be 1 or 2");
    if (b->order_bytes == 1 && 4 * I->m > 256) return fail(PS_ERR_RANGE, "uint8 op codes need m <= 64");
    if ((uintptr_t)b->stage_orders & 7u) return fail(PS_ERR_INVALID, "stage_orders must be 8-byte aligned");
    if ((r->trace_code != nullptr) != (r->trace_start != nullptr))
        return fail(PS_ERR_INVALID, "trace_code and trace_start go together");
    if (r->trace_code && r->trace_stride < 5 * I->P * I->m)
        return fail(PS_ERR_INVALID, "trace_stride %d < 5*P*m", r->trace_stride);
    DeviceGuard guard(I->device);
    if (!guard.ok) return fail(PS_ERR_CUDA, "cannot select device %d", I->device);
    EvalParams p;
    memset(&p, 0, sizeof p);
    fill_instance(I, &p);
    p.N = b->num_candidates;
    p.orders = b->stage_orders;
    p.order_u8 = b->order_bytes == 1;
    p.masks = b->offload_mask;
    p.chorders = b->channel_orders;
    p.chan_stride = b->chan_stride;
    p.makespan = r->makespan;
    p.bubble = r->bubble;
    p.peak = r->peak;
    p.flags = r->flags;
    p.blocked = r->blocked;
    p.tcode = r->trace_code;
    p.tstart = r->trace_start;
    p.tstride = r->trace_stride;
    p.events_total = (unsigned long long *)r->events_total;
    p.ready = ready;
    p.ready_chunk = ready_chunk;
    int rc = run_eval(I, p, false, stream, b->base, first_list);
    if (rc) return rc;
    // Rows that are not permutations (the evaluator flags them malformed) are replayed with the
    // reference's literal semantics: they end in OrderInfeasible with its blocked stages
    // (ps_literal.cu).  Scratch for up to 1024 concurrent replays, at most 128 MiB.
    const size_t slot = literal_slot_bytes(I->P, I->m, I->G);
    const int slots = (int)std::max<int64_t>(1, std::min<int64_t>({p.N, 1024, (int64_t)((128u << 20) / slot)}));
    int64_t *scratch = nullptr;
    PS_CUDA(cudaMallocAsync((void **)&scratch, (size_t)slots * slot, stream));
    cudaError_t e = literal_launch(p, I->v64, scratch, slots, stream);
    if (e != cudaSuccess) return cuda_fail(e, "literal replay launch");
    PS_CUDA(cudaFreeAsync(scratch, stream));
    return PS_OK;
}

// ---- delta-encoded host batches: rebuild full candidates in HBM -------------------------------

// One warp per (candidate, stage): copy the reference row; the stage-0 warp copies the mask.
__global__ void delta_rows_kernel(int64_t N, int P, int stride, int mask_words, const uint16_t *ref,
                                  const uint32_t *ref_mask, uint16_t *out, uint32_t *out_mask,
                                  const unsigned long long *moves) {
    // one warp per candidate (only the general ones are rebuilt; the rest are evaluated as moves)
    const int64_t c = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (c >= N) return;
    if (moves && unpack_move(moves[c]).type != MOVE_GENERAL) return;
    const uint32_t *src = reinterpret_cast<const uint32_t *>(ref);
    uint32_t *dst = reinterpret_cast<uint32_t *>(out + (size_t)c * P * stride);
    for (int q = lane; q < P * stride / 2; q += 32) dst[q] = src[q];
    for (int w = lane; w < mask_words; w += 32) out_mask[(size_t)c * mask_words + w] = ref_mask[w];
}

// One thread per candidate: apply its differences (after delta_rows_kernel, same stream).
__global__ void delta_apply_kernel(int64_t N, int P, int stride, int mask_words, const uint32_t *doff,
                                   const uint32_t *diffs, const uint32_t *foff, const uint32_t *flips,
                                   uint16_t *out, uint32_t *out_mask, const unsigned long long *moves) {
    const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= N) return;
    if (moves && unpack_move(moves[c]).type != MOVE_GENERAL) return;
    for (uint32_t k = doff[c]; k < doff[c + 1]; ++k) {
        const uint32_t e = diffs[2 * (size_t)k];
        out[((size_t)c * P + (e >> 16)) * stride + (e & 0xFFFFu)] = (uint16_t)diffs[2 * (size_t)k + 1];
    }
    for (uint32_t k = foff[c]; k < foff[c + 1]; ++k) {
        const uint32_t b = flips[k];
        out_mask[(size_t)c * mask_words + (b >> 5)] ^= 1u << (b & 31);
    }
}

// Classify each delta-encoded candidate: one move of the reference structure —
// SHIFT (the diffs are one stage's contiguous run of positions holding the reference run rotated by
// one: the op at one end moved to the other), TOGGLE (one offloadable bit flipped) or NOOP — is
// evaluated by the move-encoded search kernel against the reference (and its recorded base);
// anything else is GENERAL (rebuilt in HBM and evaluated materialised), INVALID when an entry is
// out of range (the call then fails).
__global__ void delta_classify_kernel(MoveCtx c, int64_t N, uint64_t nd, uint64_t nf, int moves_ok,
                                      const uint16_t *ref, const uint32_t *doff, const uint32_t *diffs,
                                      const uint32_t *foff, const uint32_t *flips, unsigned long long *moves,
                                      int32_t *general, int32_t *err) {
    const int64_t n = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (n >= N) return;
    const uint32_t d0 = doff[n], d1 = doff[n + 1], f0 = foff[n], f1 = foff[n + 1];
    Move mv;
    mv.type = MOVE_GENERAL;
    mv.stage = mv.a = mv.b = mv.mb = 0;
    bool ok = d0 <= d1 && d1 <= nd && f0 <= f1 && f1 <= nf;
    for (uint32_t k = d0; ok && k < d1; ++k) {
        const uint32_t e = diffs[2 * (size_t)k];
        if ((int)(e >> 16) >= c.P || (int)(e & 0xFFFFu) >= c.L) ok = false;
    }
    for (uint32_t k = f0; ok && k < f1; ++k)
        if (flips[k] >= (uint32_t)(c.P * c.m)) ok = false;
    if (!ok) {
        mv.type = MOVE_INVALID;
        atomicOr(err, 1);
    } else if (moves_ok) {
        const uint32_t nd_c = d1 - d0, nf_c = f1 - f0;
        if (nd_c == 0 && nf_c == 0) {
            mv.type = MOVE_NOOP;
        } else if (nd_c == 0 && nf_c == 1) {
            const int s = (int)(flips[f0] / (uint32_t)c.m), j = (int)(flips[f0] % (uint32_t)c.m);
            if (ctx_offloadable(c, s, j)) { mv.type = MOVE_TOGGLE; mv.stage = s; mv.mb = j; }
        } else if (nf_c == 0 && nd_c >= 2) {
            const uint32_t e0 = diffs[2 * (size_t)d0];
            const int s = (int)(e0 >> 16), lo = (int)(e0 & 0xFFFFu), hi = lo + (int)nd_c - 1;
            bool run = hi < c.L;
            for (uint32_t t = 0; run && t < nd_c; ++t) {
                const uint32_t e = diffs[2 * (size_t)(d0 + t)];
                run = (int)(e >> 16) == s && (int)(e & 0xFFFFu) == lo + (int)t;
            }
            if (run) {
                const uint16_t *row = ref + (size_t)s * c.stride;
                bool left = true, right = true;
                for (uint32_t t = 0; t < nd_c; ++t) {
                    const uint32_t code = diffs[2 * (size_t)(d0 + t) + 1];
                    left = left && code == (uint32_t)(t + 1 < nd_c ? row[lo + t + 1] : row[lo]);
                    right = right && code == (uint32_t)(t > 0 ? row[lo + t - 1] : row[hi]);
                }
                if (left || right) {
                    mv.type = MOVE_SHIFT;
                    mv.stage = s;
                    mv.a = left ? lo : hi;
                    mv.b = left ? hi : lo;
                }
            }
        }
    }
    moves[n] = pack_move(mv);
    if (mv.type == MOVE_GENERAL) general[1 + atomicAdd(general, 1)] = (int32_t)n;
}

// *flag = 0 if the two structures differ (the recorded base is not the delta batch's reference).
__global__ void same_structure_kernel(const uint16_t *a, const uint16_t *b, int n16, const uint32_t *ma,
                                      const uint32_t *mb, int nm, int32_t *flag) {
    for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < n16; k += gridDim.x * blockDim.x)
        if (a[k] != b[k]) *flag = 0;
    for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < nm; k += gridDim.x * blockDim.x)
        if (ma[k] != mb[k]) *flag = 0;
}

// The reference structure is a valid one (each stage row a permutation of its 3m ops), so its
// moves need no validation.
static bool valid_structure(const ps_instance *I, const uint16_t *ref) {
    std::vector<unsigned char> seen((size_t)I->m * 3);
    for (int i = 0; i < I->P; ++i) {
        std::fill(seen.begin(), seen.end(), 0);
        for (int q = 0; q < I->L; ++q) {
            const uint32_t op = ref[(size_t)i * I->stride + q], j = op >> 2, k = op & 3u;
            if (j >= (uint32_t)I->m || k > 2u || seen[j * 3 + k]) return false;
            seen[j * 3 + k] = 1;
        }
    }
    return true;
}

bool moves_incumbent_fits(const ps_instance *I);

int ps_eval_batch_host_delta(const ps_instance *I, const ps_delta_batch *b, const ps_result_batch *r, void *stream) {
    NvtxRange nvtx("ps_eval_batch_host_delta n=%llu", (unsigned long long)(b ? b->num_candidates : 0));
    if (!I || !b || !r) return fail(PS_ERR_INVALID, "null argument");
    const int64_t N = b->num_candidates;
    if (N <= 0) return N == 0 ? PS_OK : fail(PS_ERR_INVALID, "negative candidate count");
    if (!b->ref_orders || !b->ref_mask || !b->diff_offset || !b->flip_offset)
        return fail(PS_ERR_INVALID, "ref_orders, ref_mask, diff_offset and flip_offset are required");
    if (r->events_total) return fail(PS_ERR_INVALID, "events_total is a device counter: use ps_eval_batch");
    const uint64_t nd = b->diff_offset[N], nf = b->flip_offset[N];
    if ((nd && !b->diffs) || (nf && !b->flips)) return fail(PS_ERR_INVALID, "diffs / flips missing");
    if (nd > 0xFFFFFFFFull || nf > 0xFFFFFFFFull) return fail(PS_ERR_RANGE, "at most 2^32-1 diffs and flips");
    DeviceGuard guard(I->device);
    if (!guard.ok) return fail(PS_ERR_CUDA, "cannot select device %d", I->device);
    cudaStream_t s = (cudaStream_t)stream;
    // Candidates that are one move of the reference run on the move-encoded kernel (as search
    // rounds do), when the reference is well formed, its incumbent copy fits in shared memory and no
    // time can leave the evaluator's range (PS_FLAG_RANGE candidates need rows for the 64-bit pass).
    const bool moves_ok = env_int("PS_DELTA_MOVES", 1) != 0 && I->time_safe == INT_MAX &&
                          moves_incumbent_fits(I) && valid_structure(I, b->ref_orders);
    // device arena: the encoded batch, the move list, the general list and flags, the rebuilt
    // candidates, the outputs
    const size_t n_ref = (size_t)I->P * I->stride * 2, n_rmask = (size_t)I->mask_words * 4;
    const size_t n_off = (size_t)(N + 1) * 4, n_diff = (size_t)nd * 8, n_flip = (size_t)nf * 4;
    const size_t n_ord = (size_t)N * I->P * I->stride * 2, n_mask = (size_t)N * I->mask_words * 4;
    const size_t n_peak = r->peak ? (size_t)N * I->P * 8 : 0, n_blk = r->blocked ? (size_t)N * 4 : 0;
    enum { A_REF, A_RMASK, A_DOFF, A_DIFF, A_FOFF, A_FLIP, A_ORD, A_MASK, A_SPAN, A_BUB, A_PEAK, A_FLAGS, A_BLK,
           A_MOVES, A_GEN, A_FLAG2, A_COUNT };
    size_t sizes[A_COUNT] = {n_ref, n_rmask, n_off, n_diff, n_off, n_flip, n_ord, n_mask, (size_t)N * 8, (size_t)N * 8,
                             n_peak, (size_t)N * 4, n_blk, (size_t)N * 8, (size_t)(N + 1) * 4, 8};
    size_t off[A_COUNT], total = 0;
    for (int k = 0; k < A_COUNT; ++k) { off[k] = total; total += (sizes[k] + 255) & ~(size_t)255; }
    char *arena = nullptr;
    PS_CUDA(cudaMallocAsync((void **)&arena, total, s));
    const void *srcs[6] = {b->ref_orders, b->ref_mask, b->diff_offset, b->diffs, b->flip_offset, b->flips};
    for (int k = 0; k < 6; ++k)
        if (sizes[k]) PS_CUDA(cudaMemcpyAsync(arena + off[k], srcs[k], sizes[k], cudaMemcpyHostToDevice, s));
    const uint16_t *ref_d = (const uint16_t *)(arena + off[A_REF]);
    const uint32_t *rmask_d = (const uint32_t *)(arena + off[A_RMASK]);
    unsigned long long *moves = (unsigned long long *)(arena + off[A_MOVES]);
    int32_t *general = (int32_t *)(arena + off[A_GEN]);
    int32_t *flags2 = (int32_t *)(arena + off[A_FLAG2]);       // [0] error, [1] base is the reference
    PS_CUDA(cudaMemsetAsync(general, 0, 4, s));
    const int32_t init2[2] = {0, 1};
    PS_CUDA(cudaMemcpyAsync(flags2, init2, 8, cudaMemcpyHostToDevice, s));
    delta_classify_kernel<<<(unsigned)((N + 255) / 256), 256, 0, s>>>(
        move_ctx(I), N, nd, nf, moves_ok ? 1 : 0, ref_d, (const uint32_t *)(arena + off[A_DOFF]),
        (const uint32_t *)(arena + off[A_DIFF]), (const uint32_t *)(arena + off[A_FOFF]),
        (const uint32_t *)(arena + off[A_FLIP]), moves, general, flags2);
    PS_CUDA(cudaGetLastError());
    const ps_base *B = b->base && b->base->inst == I ? b->base : nullptr;
    if (B && moves_ok) {
        same_structure_kernel<<<32, 256, 0, s>>>(ref_d, B->orders, I->P * I->stride, rmask_d, B->mask, I->mask_words,
                                                 flags2 + 1);
        PS_CUDA(cudaGetLastError());
    }
    ps_result_batch dr = *r;
    dr.makespan = (int64_t *)(arena + off[A_SPAN]);
    dr.bubble = (double *)(arena + off[A_BUB]);
    dr.peak = n_peak ? (int64_t *)(arena + off[A_PEAK]) : nullptr;
    dr.flags = (uint32_t *)(arena + off[A_FLAGS]);
    dr.blocked = n_blk ? (uint32_t *)(arena + off[A_BLK]) : nullptr;
    dr.trace_code = nullptr;
    dr.trace_start = nullptr;
    dr.trace_stride = 0;
    int rc = PS_OK;
    if (moves_ok) {
        // pass 1: the move candidates (GENERAL / INVALID ones are skipped by the kernel)
        EvalParams p;
        memset(&p, 0, sizeof p);
        fill_instance(I, &p);
        p.N = N;
        p.inc_orders = ref_d;
        p.inc_mask = rmask_d;
        p.move_list = moves;
        p.base_valid = B ? flags2 + 1 : nullptr;
        p.shift_permille = 1000;
        p.max_shift = 1;
        p.makespan = dr.makespan;
        p.bubble = dr.bubble;
        p.peak = dr.peak;
        p.flags = dr.flags;
        p.blocked = dr.blocked;
        rc = run_eval(I, p, true, s, B);
    }
    if (rc == PS_OK) {
        // pass 2: the general candidates, rebuilt in HBM and evaluated materialised
        uint16_t *ord = (uint16_t *)(arena + off[A_ORD]);
        uint32_t *msk = (uint32_t *)(arena + off[A_MASK]);
        const int64_t warps = N;
        delta_rows_kernel<<<(unsigned)((warps * 32 + 255) / 256), 256, 0, s>>>(
            N, I->P, I->stride, I->mask_words, ref_d, rmask_d, ord, msk, moves);
        delta_apply_kernel<<<(unsigned)((N + 127) / 128), 128, 0, s>>>(
            N, I->P, I->stride, I->mask_words, (const uint32_t *)(arena + off[A_DOFF]),
            (const uint32_t *)(arena + off[A_DIFF]), (const uint32_t *)(arena + off[A_FOFF]),
            (const uint32_t *)(arena + off[A_FLIP]), ord, msk, moves);
        PS_CUDA(cudaGetLastError());
        ps_cand_batch db;
        memset(&db, 0, sizeof db);
        db.num_candidates = N;
        db.stage_orders = ord;
        db.offload_mask = msk;
        db.base = b->base;
        db.order_bytes = 2;
        rc = eval_batch_impl(I, &db, &dr, s, nullptr, 0, general);
    }
    int32_t h_err = 0;
    if (rc == PS_OK) {
        PS_CUDA(cudaMemcpyAsync(r->makespan, dr.makespan, (size_t)N * 8, cudaMemcpyDeviceToHost, s));
        PS_CUDA(cudaMemcpyAsync(r->bubble, dr.bubble, (size_t)N * 8, cudaMemcpyDeviceToHost, s));
        PS_CUDA(cudaMemcpyAsync(r->flags, dr.flags, (size_t)N * 4, cudaMemcpyDeviceToHost, s));
        if (n_peak) PS_CUDA(cudaMemcpyAsync(r->peak, dr.peak, n_peak, cudaMemcpyDeviceToHost, s));
        if (n_blk) PS_CUDA(cudaMemcpyAsync(r->blocked, dr.blocked, n_blk, cudaMemcpyDeviceToHost, s));
        PS_CUDA(cudaMemcpyAsync(&h_err, flags2, 4, cudaMemcpyDeviceToHost, s));
    }
    cudaFreeAsync(arena, s);
    cudaError_t e = cudaStreamSynchronize(s);
    if (rc) return rc;
    if (e != cudaSuccess) return cuda_fail(e, "ps_eval_batch_host_delta");
    if (h_err) return fail(PS_ERR_INVALID, "a diff or flip entry (or offset) is out of range");
    return PS_OK;
}

// Pinned host word holding 1: the copy engine writes it behind each chunk as its ready flag.
static const int32_t *pinned_one() {
    static int32_t *one = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        if (cudaHostAlloc((void **)&one, sizeof(int32_t), cudaHostAllocPortable) == cudaSuccess) *one = 1;
        else one = nullptr;
    });
    return one;
}

int ps_eval_batch_host(const ps_instance *I, const ps_cand_batch *b, const ps_result_batch *r, void *stream) {
    NvtxRange nvtx("ps_eval_batch_host n=%llu", (unsigned long long)(b ? b->num_candidates : 0));
    if (!I || !b || !r) return fail(PS_ERR_INVALID, "null argument");
    const int64_t N = b->num_candidates;
    if (N <= 0) return N == 0 ? PS_OK : fail(PS_ERR_INVALID, "negative candidate count");
    if (!b->stage_orders || !b->offload_mask) return fail(PS_ERR_INVALID, "stage_orders and offload_mask are required");
    if (r->events_total) return fail(PS_ERR_INVALID, "events_total is a device counter: use ps_eval_batch");
    if (b->order_bytes != 0 && b->order_bytes != 1 && b->order_bytes != 2)
        return fail(PS_ERR_INVALID, "order_bytes must be 1 or 2");
    const int ob = b->order_bytes == 1 ? 1 : 2;
    if (ob == 1 && 4 * I->m > 256) return fail(PS_ERR_RANGE, "uint8 op codes need m <= 64");
    DeviceGuard guard(I->device);
    if (!guard.ok) return fail(PS_ERR_CUDA, "cannot select device %d", I->device);
    const int32_t *one = pinned_one();
    if (!one) return fail(PS_ERR_NOMEM, "pinned flag word");
    cudaStream_t s = (cudaStream_t)stream;
    // Inputs stream in over PCIe in chunks on a copy stream while ONE evaluation launch runs: the
    // copy engine writes a ready flag behind each chunk and warps wait for their candidate's flag
    // (candidates are taken in index order), so copy and evaluation overlap without wave tails.
    const int64_t chunk = std::max<int64_t>(1, env_int("PS_HOST_CHUNK", 4096));
    const int nchunks = (int)((N + chunk - 1) / chunk);
    const size_t n_ord = (size_t)N * I->P * I->stride * ob, n_mask = (size_t)N * I->mask_words * 4;
    const size_t n_chan = b->channel_orders ? (size_t)N * I->G * b->chan_stride * 4 : 0;
    const size_t n_peak = r->peak ? (size_t)N * I->P * 8 : 0;
    const size_t n_tr = r->trace_code ? (size_t)N * r->trace_stride * 4 : 0;
    const size_t n_blk = r->blocked ? (size_t)N * 4 : 0;
    // one device arena: inputs, ready flags, outputs
    size_t off[11], total = 0;
    size_t sizes[11] = {n_ord, n_mask, n_chan, (size_t)nchunks * 4, (size_t)N * 8, (size_t)N * 8, n_peak,
                        (size_t)N * 4, n_blk, n_tr, n_tr};
    for (int k = 0; k < 11; ++k) { off[k] = total; total += (sizes[k] + 255) & ~(size_t)255; }
    char *arena = nullptr;
    PS_CUDA(cudaMallocAsync((void **)&arena, total, s));
    int32_t *ready = (int32_t *)(arena + off[3]);
    PS_CUDA(cudaMemsetAsync(ready, 0, (size_t)nchunks * 4, s));
    // the copy stream and its two events are kept per thread and device
    struct CopyRes { cudaStream_t cs = nullptr; cudaEvent_t start = nullptr, copied = nullptr; };
    static thread_local std::map<int, CopyRes> copy_res;
    CopyRes &cr = copy_res[I->device];
    if (!cr.cs) {
        PS_CUDA(cudaStreamCreateWithFlags(&cr.cs, cudaStreamNonBlocking));
        PS_CUDA(cudaEventCreateWithFlags(&cr.start, cudaEventDisableTiming));
        PS_CUDA(cudaEventCreateWithFlags(&cr.copied, cudaEventDisableTiming));
    }
    cudaStream_t cs = cr.cs;
    cudaEvent_t ev_start = cr.start, ev_copied = cr.copied;
    PS_CUDA(cudaEventRecord(ev_start, s));                  // arena and cleared flags exist
    PS_CUDA(cudaStreamWaitEvent(cs, ev_start, 0));
    // every copy is enqueued before the evaluation launches: the flags it waits for are certain
    const size_t ord_row = (size_t)I->P * I->stride * ob, mask_row = (size_t)I->mask_words * 4;
    const size_t chan_row = b->channel_orders ? (size_t)I->G * b->chan_stride * 4 : 0;
    for (int c = 0; c < nchunks; ++c) {
        const int64_t lo = c * chunk, n = std::min(chunk, N - lo);
        PS_CUDA(cudaMemcpyAsync(arena + off[0] + lo * ord_row, (const char *)b->stage_orders + lo * ord_row,
                                n * ord_row, cudaMemcpyHostToDevice, cs));
        PS_CUDA(cudaMemcpyAsync(arena + off[1] + lo * mask_row, (const char *)b->offload_mask + lo * mask_row,
                                n * mask_row, cudaMemcpyHostToDevice, cs));
        if (n_chan)
            PS_CUDA(cudaMemcpyAsync(arena + off[2] + lo * chan_row, (const char *)b->channel_orders + lo * chan_row,
                                    n * chan_row, cudaMemcpyHostToDevice, cs));
        PS_CUDA(cudaMemcpyAsync(ready + c, one, sizeof(int32_t), cudaMemcpyHostToDevice, cs));
    }
    PS_CUDA(cudaEventRecord(ev_copied, cs));
    ps_cand_batch db = *b;
    db.stage_orders = arena + off[0];
    db.offload_mask = (const uint32_t *)(arena + off[1]);
    db.channel_orders = n_chan ? (const uint32_t *)(arena + off[2]) : nullptr;
    ps_result_batch dr = *r;
    dr.makespan = (int64_t *)(arena + off[4]);
    dr.bubble = (double *)(arena + off[5]);
    dr.peak = n_peak ? (int64_t *)(arena + off[6]) : nullptr;
    dr.flags = (uint32_t *)(arena + off[7]);
    dr.blocked = n_blk ? (uint32_t *)(arena + off[8]) : nullptr;
    dr.trace_code = n_tr ? (uint32_t *)(arena + off[9]) : nullptr;
    dr.trace_start = n_tr ? (int32_t *)(arena + off[10]) : nullptr;
    int rc = eval_batch_impl(I, &db, &dr, s, ready, chunk);
    cudaStreamWaitEvent(s, ev_copied, 0);
    if (rc == PS_OK) {
        PS_CUDA(cudaMemcpyAsync(r->makespan, dr.makespan, (size_t)N * 8, cudaMemcpyDeviceToHost, s));
        PS_CUDA(cudaMemcpyAsync(r->bubble, dr.bubble, (size_t)N * 8, cudaMemcpyDeviceToHost, s));
        PS_CUDA(cudaMemcpyAsync(r->flags, dr.flags, (size_t)N * 4, cudaMemcpyDeviceToHost, s));
        if (n_peak) PS_CUDA(cudaMemcpyAsync(r->peak, dr.peak, n_peak, cudaMemcpyDeviceToHost, s));
        if (n_blk) PS_CUDA(cudaMemcpyAsync(r->blocked, dr.blocked, n_blk, cudaMemcpyDeviceToHost, s));
        if (n_tr) {
            PS_CUDA(cudaMemcpyAsync(r->trace_code, dr.trace_code, n_tr, cudaMemcpyDeviceToHost, s));
            PS_CUDA(cudaMemcpyAsync(r->trace_start, dr.trace_start, n_tr, cudaMemcpyDeviceToHost, s));
        }
    }
    cudaFreeAsync(arena, s);
    cudaError_t e = cudaStreamSynchronize(s);
    cudaStreamSynchronize(cs);
    if (rc) return rc;
    if (e != cudaSuccess) return cuda_fail(e, "ps_eval_batch_host");
    return PS_OK;
}

extern "C" cudaError_t ps_bound_launch(int P, int m, int uniform, int post, int comm, const int32_t *proc, int64_t N,
                            const int32_t *clock, const int32_t *sfree, const int32_t *start, int64_t *lb,
                            int num_sms, cudaStream_t s);

int ps_bound_batch_eval(const ps_instance *I, const ps_bound_batch *b, int64_t *lower_bound, void *stream) {
    NvtxRange nvtx("ps_bound_batch_eval");
    if (!I || !b || !lower_bound) return fail(PS_ERR_INVALID, "null argument");
    if (b->num_nodes < 0) return fail(PS_ERR_INVALID, "negative node count");
    if (b->num_nodes == 0) return PS_OK;
    if (!b->clock || !b->stage_free || !b->comp_start) return fail(PS_ERR_INVALID, "clock, stage_free and comp_start are required");
    DeviceGuard guard(I->device);
    if (!guard.ok) return fail(PS_ERR_CUDA, "cannot select device %d", I->device);
    cudaError_t e = ps_bound_launch(I->P, I->m, I->uniform, I->post, I->comm, I->d_proc, b->num_nodes, b->clock,
                                    b->stage_free, b->comp_start, lower_bound, I->num_sms, (cudaStream_t)stream);
    if (e != cudaSuccess) return cuda_fail(e, "bound launch");
    return PS_OK;
}

// The move-encoded kernels keep the incumbent in shared memory, with one warp's bitsets behind it.
bool moves_incumbent_fits(const ps_instance *I) {
    return (size_t)(incumbent_words(I, true) + ((3 * I->P * I->MW + 3) & ~3)) * 4 <= (size_t)I->max_smem_optin;
}

__global__ void best_key_kernel(const int64_t *span, const uint32_t *flags, int64_t n, int64_t first, long long *best);

// A search round for an incumbent too large for shared memory (P = 32 with m above ~1,100): the
// neighbours are materialised in chunks and evaluated as rows (with prefix sharing against the
// recorded base), each chunk's best key folded into *best_key — the same key as the move-encoded
// round (a duplicate move only costs its own evaluation).
int search_round_rows(const ps_instance *I, const ps_search_desc *d, int64_t *best_key, int64_t *makespan_out,
                      cudaStream_t s) {
    const size_t per = (size_t)I->P * I->stride * 2 + (size_t)I->mask_words * 4 + 8 + 8 + 4;
    const int64_t cap = std::max<int64_t>(256, (int64_t)(((size_t)env_int("PS_ROWS_CHUNK_MB", 2048) << 20) / per));
    const int64_t chunk = std::min<int64_t>(d->count, std::min<int64_t>(cap, 16384));
    char *arena = nullptr;
    PS_CUDA(cudaMallocAsync((void **)&arena, (size_t)chunk * per + 5 * 256, s));
    size_t off = 0;
    auto take = [&](size_t n) { char *q = arena + off; off += (n + 255) & ~(size_t)255; return q; };
    uint16_t *ord = (uint16_t *)take((size_t)chunk * I->P * I->stride * 2);
    uint32_t *msk = (uint32_t *)take((size_t)chunk * I->mask_words * 4);
    int64_t *span = (int64_t *)take((size_t)chunk * 8);
    double *bub = (double *)take((size_t)chunk * 8);
    uint32_t *flg = (uint32_t *)take((size_t)chunk * 4);
    int rc = PS_OK;
    for (int64_t lo = 0; lo < d->count && rc == PS_OK; lo += chunk) {
        const int64_t n = std::min(chunk, d->count - lo);
        materialize_kernel<<<(unsigned)((n * I->P * 32 + 255) / 256), 256, 0, s>>>(
            move_ctx(I), d->moves, d->round, d->first_index + lo, n, d->inc_orders, d->inc_mask, ord, msk);
        cudaError_t e = cudaGetLastError();
        if (e != cudaSuccess) { rc = cuda_fail(e, "materialize"); break; }
        EvalParams p;
        memset(&p, 0, sizeof p);
        fill_instance(I, &p);
        p.N = n;
        p.orders = ord;
        p.masks = msk;
        p.makespan = makespan_out ? makespan_out + lo : span;
        p.bubble = bub;
        p.flags = flg;
        p.events_total = (unsigned long long *)d->events_total;
        if ((rc = run_eval(I, p, false, s, d->base)) != PS_OK) break;
        best_key_kernel<<<std::max(1, std::min((int)((n + 255) / 256), 4 * I->num_sms)), 256, 0, s>>>(
            p.makespan, flg, n, d->first_index + lo, (long long *)best_key);
        if ((e = cudaGetLastError()) != cudaSuccess) rc = cuda_fail(e, "best key");
    }
    cudaFreeAsync(arena, s);
    return rc;
}

int ps_search_round(const ps_instance *I, const ps_search_desc *d, int64_t *best_key, int64_t *makespan_out,
                    void *stream) {
    NvtxRange nvtx("ps_search_round r=%llu", (unsigned long long)(d ? d->round : 0));
    if (!I || !d || !best_key) return fail(PS_ERR_INVALID, "null argument");
    if (!d->inc_orders || !d->inc_mask) return fail(PS_ERR_INVALID, "incumbent buffers are required");
    if (d->count < 0 || d->first_index < 0) return fail(PS_ERR_INVALID, "negative shard range");
    if ((uint64_t)(d->first_index + d->count) > 0xFFFFFFFFull)
        return fail(PS_ERR_RANGE, "neighbour indices must stay below 2^32");
    if (d->moves.shift_permille > 1000u || d->moves.max_shift < 1u)
        return fail(PS_ERR_INVALID, "shift_permille must be <= 1000 and max_shift >= 1");
    DeviceGuard guard(I->device);
    if (!guard.ok) return fail(PS_ERR_CUDA, "cannot select device %d", I->device);
    EvalParams p;
    memset(&p, 0, sizeof p);
    fill_instance(I, &p);
    p.N = d->count;
    p.inc_orders = d->inc_orders;
    p.inc_mask = d->inc_mask;
    p.seed = d->moves.seed;
    p.round = d->round;
    p.first_index = d->first_index;
    p.shift_permille = d->moves.shift_permille;
    p.max_shift = d->moves.max_shift;
    p.makespan = makespan_out;
    p.best_key = (long long *)best_key;
    p.dedup = makespan_out == nullptr && d->dedup;
    // (bound pruning sums a stage's remaining work in 32 bits: only where the horizon fits them)
    p.cutoff = makespan_out == nullptr && d->cutoff > 0 && I->time_safe == INT_MAX ? d->cutoff : 0;
    p.events_total = (unsigned long long *)d->events_total;
    if (!moves_incumbent_fits(I) || env_int("PS_SEARCH_ROWS", 0) != 0) {     // (the knob: tests)
        if (d->count == 0) return PS_OK;
        return search_round_rows(I, d, best_key, makespan_out, (cudaStream_t)stream);
    }
    return run_eval(I, p, true, (cudaStream_t)stream, d->base);
}

// ---- channel-order search: explicit channel orders, reload/offload shifts ----

struct XMove {
    int type;          // 0 no-op, 1 stage-op SHIFT, 3 transfer RSHIFT
    int row, a, b;     // stage (SHIFT) or channel (RSHIFT); element at a moves to b
};

// lens[g] = transfers in the incumbent's channel g (entries before the first pad), lens[G] = total.
__global__ void chan_lens_kernel(const uint32_t *inc_chan, int G, int cstride, int *lens) {
    __shared__ int tot;
    if (threadIdx.x == 0) tot = 0;
    __syncthreads();
    for (int g = threadIdx.x; g < G; g += blockDim.x) {
        int n = 0;
        while (n < cstride && inc_chan[(size_t)g * cstride + n] != 0xFFFFFFFFu) ++n;
        lens[g] = n;
        atomicAdd(&tot, n);
    }
    __syncthreads();
    if (threadIdx.x == 0) lens[G] = tot;
}

// The move of neighbour `index` (oracle/ps_oracle.c or_neighbour_explicit restates it).
__device__ XMove decode_xmove(const ps_move_params &mp, uint64_t round, uint64_t index, int P, int L, int G,
                              const int *lens) {
    Philox4 r = philox4x32_10((uint32_t)index, (uint32_t)(index >> 32), (uint32_t)round, (uint32_t)(round >> 32),
                              (uint32_t)mp.seed, (uint32_t)(mp.seed >> 32));
    const uint32_t D = mp.max_shift ? mp.max_shift : 1u;
    XMove mv;
    mv.type = 0;
    mv.a = mv.b = 0;
    int n;
    const bool stage_move = lens[G] == 0 || r.v[0] % 1000u < mp.shift_permille;
    if (stage_move) {
        mv.row = (int)(r.v[1] % (uint32_t)P);
        n = L;
    } else {
        mv.row = (int)(r.v[1] % (uint32_t)G);
        n = lens[mv.row];
        if (n < 2) return mv;
    }
    const int a = (int)(r.v[2] % (uint32_t)n);
    const int d = 1 + (int)((r.v[3] >> 1) % D);
    int b = (r.v[3] & 1u) ? a - d : a + d;
    b = b < 0 ? 0 : (b > n - 1 ? n - 1 : b);
    mv.a = a;
    mv.b = b;
    if (b != a) mv.type = stage_move ? 1 : 3;
    return mv;
}

// One warp per (neighbour, row): rows [0, P) are stage orders, [P, P + G) channel orders; the
// stage-0 warp also writes the (unchanged) offload mask.
__global__ void materialize_x_kernel(MoveCtx c, ps_move_params mp, uint64_t round, int64_t first, int64_t count,
                                     int G, int cstride, const int *lens, const uint16_t *inc,
                                     const uint32_t *inc_mask, const uint32_t *inc_chan, uint16_t *out,
                                     uint32_t *out_mask, uint32_t *out_chan) {
    const int64_t row = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    const int R = c.P + G;
    if (row >= count * R) return;
    const int64_t n = row / R;
    const int r = (int)(row % R);
    const XMove mv = decode_xmove(mp, round, (uint64_t)(first + n), c.P, c.L, G, lens);
    if (r < c.P) {
        const bool sh = mv.type == 1 && mv.row == r;
        const uint16_t *src = inc + (size_t)r * c.stride;
        uint16_t *dst = out + ((size_t)n * c.P + r) * c.stride;
        for (int q = lane; q < c.stride; q += 32)
            dst[q] = q < c.L ? src[sh ? shifted_position(q, mv.a, mv.b) : q] : (uint16_t)0;
        if (r == 0)
            for (int w = lane; w < c.mask_words; w += 32) out_mask[(size_t)n * c.mask_words + w] = inc_mask[w];
    } else {
        const int g = r - c.P;
        const bool sh = mv.type == 3 && mv.row == g;
        const uint32_t *src = inc_chan + (size_t)g * cstride;
        uint32_t *dst = out_chan + ((size_t)n * G + g) * cstride;
        for (int q = lane; q < cstride; q += 32) dst[q] = src[sh && q < lens[g] ? shifted_position(q, mv.a, mv.b) : q];
    }
}

__global__ void apply_x_kernel(MoveCtx c, ps_move_params mp, uint64_t round, uint64_t index, int G, int cstride,
                               const int *lens, uint16_t *inc, uint32_t *inc_chan) {
    if (threadIdx.x) return;
    const XMove mv = decode_xmove(mp, round, index, c.P, c.L, G, lens);
    if (mv.type == 1) {
        uint16_t *row = inc + (size_t)mv.row * c.stride;
        const uint16_t v = row[mv.a];
        if (mv.a < mv.b) for (int q = mv.a; q < mv.b; ++q) row[q] = row[q + 1];
        else for (int q = mv.a; q > mv.b; --q) row[q] = row[q - 1];
        row[mv.b] = v;
    } else if (mv.type == 3) {
        uint32_t *row = inc_chan + (size_t)mv.row * cstride;
        const uint32_t v = row[mv.a];
        if (mv.a < mv.b) for (int q = mv.a; q < mv.b; ++q) row[q] = row[q + 1];
        else for (int q = mv.a; q > mv.b; --q) row[q] = row[q - 1];
        row[mv.b] = v;
    }
}

// best_key = min over feasible neighbours of (makespan << 32 | global index)
__global__ void best_key_kernel(const int64_t *makespan, const uint32_t *flags, int64_t n, int64_t first,
                                long long *best_key) {
    long long best = LLONG_MAX;
    for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < n; k += (int64_t)gridDim.x * blockDim.x)
        if (flags[k] == FLAG_FEASIBLE) {
            const long long key = ((long long)makespan[k] << 32) | (long long)(uint32_t)(first + k);
            best = key < best ? key : best;
        }
    for (int o = 16; o; o >>= 1) {
        const long long v = __shfl_xor_sync(0xffffffffu, best, o);
        best = v < best ? v : best;
    }
    if ((threadIdx.x & 31) == 0 && best != LLONG_MAX) atomicMin(best_key, best);
}

// NCCL, resolved at run time: the library stays loadable on hosts without NCCL, and shares the
// process's libnccl.so.2 (e.g. the one torch.distributed already loaded) with the caller.
typedef ncclResult_t (*AllReduceFn)(const void *, void *, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                                    cudaStream_t);
typedef const char *(*ErrStrFn)(ncclResult_t);
static AllReduceFn nccl_allreduce(ErrStrFn *errstr) {
    static AllReduceFn fn = nullptr;
    static ErrStrFn es = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        void *h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL | RTLD_NOLOAD);
        if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
        if (h) {
            fn = (AllReduceFn)dlsym(h, "ncclAllReduce");
            es = (ErrStrFn)dlsym(h, "ncclGetErrorString");
        }
    });
    if (errstr) *errstr = es;
    return fn;
}

int ps_search_round_sharded(const ps_instance *I, const ps_search_desc *d, int64_t *best_key, int64_t *makespan_out,
                            void *nccl_comm, void *stream) {
    NvtxRange nvtx("ps_search_round_sharded");
    int rc = ps_search_round(I, d, best_key, makespan_out, stream);
    if (rc || !nccl_comm) return rc;
    ErrStrFn es = nullptr;
    AllReduceFn ar = nccl_allreduce(&es);
    if (!ar) return fail(PS_ERR_INVALID, "libnccl.so.2 not found: cannot combine the round across ranks");
    DeviceGuard guard(I->device);
    if (!guard.ok) return fail(PS_ERR_CUDA, "cannot select device %d", I->device);
    ncclResult_t r = ar(best_key, best_key, 1, ncclInt64, ncclMin, (ncclComm_t)nccl_comm, (cudaStream_t)stream);
    if (r != ncclSuccess) return fail(PS_ERR_CUDA, "ncclAllReduce: %s", es ? es(r) : "error");
    return PS_OK;
}

static int check_x(const ps_instance *I, const uint32_t *inc_chan, int chan_stride) {
    if (!inc_chan) return fail(PS_ERR_INVALID, "the incumbent's channel orders are required");
    if (chan_stride < 1) return fail(PS_ERR_INVALID, "chan_stride must be positive");
    return PS_OK;
}

int ps_materialize_moves_explicit(const ps_instance *I, const ps_search_desc *d, const uint32_t *inc_chan,
                                  int32_t chan_stride, uint16_t *orders_out, uint32_t *mask_out, uint32_t *chan_out,
                                  void *stream) {
    NvtxRange nvtx("ps_materialize_moves_explicit");
    if (!I || !d || !orders_out || !mask_out || !chan_out) return fail(PS_ERR_INVALID, "null argument");
    int rc = check_x(I, inc_chan, chan_stride);
    if (rc) return rc;
    if (d->count <= 0) return PS_OK;
    DeviceGuard guard(I->device);
    if (!guard.ok) return fail(PS_ERR_CUDA, "cannot select device %d", I->device);
    cudaStream_t s = (cudaStream_t)stream;
    int *lens = nullptr;
    PS_CUDA(cudaMallocAsync((void **)&lens, (I->G + 1) * sizeof(int), s));
    chan_lens_kernel<<<1, 32, 0, s>>>(inc_chan, I->G, chan_stride, lens);
    const int64_t warps = d->count * (I->P + I->G);
    materialize_x_kernel<<<(unsigned)((warps * 32 + 255) / 256), 256, 0, s>>>(
        move_ctx(I), d->moves, d->round, d->first_index, d->count, I->G, chan_stride, lens, d->inc_orders, d->inc_mask,
        inc_chan, orders_out, mask_out, chan_out);
    PS_CUDA(cudaGetLastError());
    PS_CUDA(cudaFreeAsync(lens, s));
    return PS_OK;
}

int ps_apply_move_explicit(const ps_instance *I, uint16_t *inc_orders, uint32_t *inc_chan, int32_t chan_stride,
                           const ps_move_params *mp, uint64_t round, uint64_t index, void *stream) {
    NvtxRange nvtx("ps_apply_move_explicit");
    if (!I || !inc_orders || !mp) return fail(PS_ERR_INVALID, "null argument");
    int rc = check_x(I, inc_chan, chan_stride);
    if (rc) return rc;
    DeviceGuard guard(I->device);
    if (!guard.ok) return fail(PS_ERR_CUDA, "cannot select device %d", I->device);
    cudaStream_t s = (cudaStream_t)stream;
    int *lens = nullptr;
    PS_CUDA(cudaMallocAsync((void **)&lens, (I->G + 1) * sizeof(int), s));
    chan_lens_kernel<<<1, 32, 0, s>>>(inc_chan, I->G, chan_stride, lens);
    apply_x_kernel<<<1, 32, 0, s>>>(move_ctx(I), *mp, round, index, I->G, chan_stride, lens, inc_orders, inc_chan);
    PS_CUDA(cudaGetLastError());
    PS_CUDA(cudaFreeAsync(lens, s));
    return PS_OK;
}

int ps_search_round_explicit(const ps_instance *I, const ps_search_desc *d, const uint32_t *inc_chan,
                             int32_t chan_stride, int64_t *best_key, int64_t *makespan_out, void *stream) {
    NvtxRange nvtx("ps_search_round_explicit r=%llu", (unsigned long long)(d ? d->round : 0));
    if (!I || !d || !best_key) return fail(PS_ERR_INVALID, "null argument");
    if (!d->inc_orders || !d->inc_mask) return fail(PS_ERR_INVALID, "incumbent buffers are required");
    int rc = check_x(I, inc_chan, chan_stride);
    if (rc) return rc;
    if (d->count < 0 || d->first_index < 0) return fail(PS_ERR_INVALID, "negative shard range");
    if ((uint64_t)(d->first_index + d->count) > 0xFFFFFFFFull)
        return fail(PS_ERR_RANGE, "neighbour indices must stay below 2^32");
    if (d->moves.shift_permille > 1000u || d->moves.max_shift < 1u)
        return fail(PS_ERR_INVALID, "shift_permille must be <= 1000 and max_shift >= 1");
    if (d->count == 0) return PS_OK;
    DeviceGuard guard(I->device);
    if (!guard.ok) return fail(PS_ERR_CUDA, "cannot select device %d", I->device);
    cudaStream_t s = (cudaStream_t)stream;
    // neighbours are materialised in chunks (stage rows + channel rows) and evaluated as an
    // explicit-channel batch; each chunk's best key folds into *best_key
    const int64_t chunk = std::min<int64_t>(d->count, std::max(256, env_int("PS_X_CHUNK", 16384)));
    const size_t ord_b = (size_t)chunk * I->P * I->stride * 2, msk_b = (size_t)chunk * I->mask_words * 4;
    const size_t chn_b = (size_t)chunk * I->G * chan_stride * 4;
    char *arena = nullptr;
    const size_t total = ord_b + msk_b + chn_b + (size_t)chunk * (8 + 8 + 4) + (I->G + 1) * 4 + 1024;
    PS_CUDA(cudaMallocAsync((void **)&arena, total, s));
    size_t off = 0;
    auto take = [&](size_t n) { char *q = arena + off; off += (n + 255) & ~(size_t)255; return q; };
    uint16_t *ord = (uint16_t *)take(ord_b);
    uint32_t *msk = (uint32_t *)take(msk_b);
    uint32_t *chn = (uint32_t *)take(chn_b);
    int64_t *span = (int64_t *)take((size_t)chunk * 8);
    double *bub = (double *)take((size_t)chunk * 8);
    uint32_t *flg = (uint32_t *)take((size_t)chunk * 4);
    int *lens = (int *)take((I->G + 1) * 4);
    (void)total;
    chan_lens_kernel<<<1, 32, 0, s>>>(inc_chan, I->G, chan_stride, lens);
    for (int64_t lo = 0; lo < d->count; lo += chunk) {
        const int64_t n = std::min(chunk, d->count - lo);
        const int64_t warps = n * (I->P + I->G);
        materialize_x_kernel<<<(unsigned)((warps * 32 + 255) / 256), 256, 0, s>>>(
            move_ctx(I), d->moves, d->round, d->first_index + lo, n, I->G, chan_stride, lens, d->inc_orders,
            d->inc_mask, inc_chan, ord, msk, chn);
        PS_CUDA(cudaGetLastError());
        EvalParams p;
        memset(&p, 0, sizeof p);
        fill_instance(I, &p);
        p.N = n;
        p.orders = ord;
        p.masks = msk;
        p.chorders = chn;
        p.chan_stride = chan_stride;
        p.makespan = makespan_out ? makespan_out + lo : span;
        p.bubble = bub;
        p.flags = flg;
        p.events_total = (unsigned long long *)d->events_total;
        rc = run_eval(I, p, false, s, d->base);   // (prefix sharing with an explicit recording of the incumbent)
        if (rc) return rc;
        best_key_kernel<<<std::max(1, std::min((int)((n + 255) / 256), 4 * I->num_sms)), 256, 0, s>>>(
            p.makespan, flg, n, d->first_index + lo, (long long *)best_key);
        PS_CUDA(cudaGetLastError());
    }
    PS_CUDA(cudaFreeAsync(arena, s));
    return PS_OK;
}

int ps_materialize_moves(const ps_instance *I, const ps_search_desc *d, uint16_t *orders_out, uint32_t *mask_out,
                         void *stream) {
    if (!I || !d || !orders_out || !mask_out) return fail(PS_ERR_INVALID, "null argument");
    if (d->count <= 0) return PS_OK;
    DeviceGuard guard(I->device);
    if (!guard.ok) return fail(PS_ERR_CUDA, "cannot select device %d", I->device);
    int64_t warps = d->count * I->P;
    int64_t blocks = (warps * 32 + 255) / 256;
    materialize_kernel<<<(unsigned)blocks, 256, 0, (cudaStream_t)stream>>>(
        move_ctx(I), d->moves, d->round, d->first_index, d->count, d->inc_orders, d->inc_mask, orders_out, mask_out);
    PS_CUDA(cudaGetLastError());
    return PS_OK;
}

int ps_apply_move(const ps_instance *I, uint16_t *inc_orders, uint32_t *inc_mask, const ps_move_params *mp,
                  uint64_t round, uint64_t index, void *stream) {
    NvtxRange nvtx("ps_apply_move");
    if (!I || !inc_orders || !inc_mask || !mp) return fail(PS_ERR_INVALID, "null argument");
    DeviceGuard guard(I->device);
    if (!guard.ok) return fail(PS_ERR_CUDA, "cannot select device %d", I->device);
    apply_move_kernel<<<1, 32, 0, (cudaStream_t)stream>>>(move_ctx(I), *mp, round, index, inc_orders, inc_mask);
    PS_CUDA(cudaGetLastError());
    return PS_OK;
}

int ps_int32_probe(int64_t iters, int64_t *lane_ops, void *stream) {
    if (!lane_ops || iters < 1) return fail(PS_ERR_INVALID, "bad probe arguments");
    int dev, sms;
    PS_CUDA(cudaGetDevice(&dev));
    PS_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    uint32_t *sink = nullptr;
    cudaStream_t s = (cudaStream_t)stream;
    PS_CUDA(cudaMallocAsync((void **)&sink, 4, s));
    int32_probe_kernel<<<sms * 8, 256, 0, s>>>(iters, 0x1234567u, (unsigned long long *)lane_ops, sink);
    PS_CUDA(cudaGetLastError());
    PS_CUDA(cudaFreeAsync(sink, s));
    return PS_OK;
}

}  // extern "C"
