// ps_eval_impl.cuh — instantiation helpers for ps_launch.h (included once per (V, MOVES) TU).
#pragma once
#include <atomic>
#include "ps_launch.h"

namespace ps {

// Raise a kernel's dynamic shared-memory limit only when a launch needs more than was already
// granted on this device (the attribute call costs microseconds on every launch otherwise).
template <typename Fn>
static cudaError_t ensure_smem(Fn fn, size_t smem, std::atomic<int> *granted) {
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    std::atomic<int> &g = granted[dev & 63];
    if ((int)smem <= g.load(std::memory_order_relaxed)) return cudaSuccess;
    e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    int cur = g.load();
    while ((int)smem > cur && !g.compare_exchange_weak(cur, (int)smem)) {}
    return cudaSuccess;
}

// one grant record per kernel instantiation and device, shared by launches and occupancy queries
template <typename V, bool MOVES, int GSTATE, bool REC, bool DERIVED, bool UNI>
static std::atomic<int> *granted_for() {
    static std::atomic<int> g[64];
    return g;
}

template <typename V, bool MOVES, int GSTATE, bool REC, bool DERIVED, bool UNI>
static cudaError_t launch_one(const EvalParams &p, LaunchCfg cfg, cudaStream_t stream) {
    auto fn = eval_kernel<V, MOVES, GSTATE, REC, DERIVED, UNI>;
    cudaError_t e = ensure_smem(fn, cfg.smem, granted_for<V, MOVES, GSTATE, REC, DERIVED, UNI>());
    if (e != cudaSuccess) return e;
    fn<<<cfg.grid, cfg.block, cfg.smem, stream>>>(p);
    return cudaGetLastError();
}

template <typename V, bool MOVES, int GSTATE, bool DERIVED, bool UNI>
static cudaError_t occ_one(int block, size_t smem, int *n) {
    auto fn = eval_kernel<V, MOVES, GSTATE, false, DERIVED, UNI>;
    cudaError_t e = ensure_smem(fn, smem, granted_for<V, MOVES, GSTATE, false, DERIVED, UNI>());
    if (e != cudaSuccess) return e;
    return cudaOccupancyMaxActiveBlocksPerMultiprocessor(n, fn, block, smem);
}

// Move-encoded candidates (the search) are always in derived channel mode; base recording is a
// single materialised candidate in derived mode with its state in shared memory.
#define PS_PICK(FN, ARGS)                                                                              \
    if (!MOVES && v.record && v.derived)                                                              \
        return v.uni ? FN<V, false, 0, true, true, true> ARGS : FN<V, false, 0, true, true, false> ARGS; \
    if (!MOVES && v.record)                                                                           \
        return v.uni ? FN<V, false, 0, true, false, true> ARGS : FN<V, false, 0, true, false, false> ARGS; \
    if (MOVES || v.derived) {                                                                         \
        if (!MOVES && v.gstate && v.nobase) return v.uni ? FN<V, MOVES, 4, false, true, true> ARGS : FN<V, MOVES, 4, false, true, false> ARGS; \
        if (v.gstate && v.wmask) return v.uni ? FN<V, MOVES, 2, false, true, true> ARGS : FN<V, MOVES, 2, false, true, false> ARGS; \
        if (v.gstate) return v.uni ? FN<V, MOVES, 1, false, true, true> ARGS : FN<V, MOVES, 1, false, true, false> ARGS; \
        if (!MOVES && v.nobase) return v.uni ? FN<V, MOVES, 3, false, true, true> ARGS : FN<V, MOVES, 3, false, true, false> ARGS; \
        return v.uni ? FN<V, MOVES, 0, false, true, true> ARGS : FN<V, MOVES, 0, false, true, false> ARGS; \
    }                                                                                                 \
    if (v.gstate && v.nobase) return v.uni ? FN<V, false, 4, false, false, true> ARGS : FN<V, false, 4, false, false, false> ARGS; \
    if (v.gstate) return v.uni ? FN<V, false, 1, false, false, true> ARGS : FN<V, false, 1, false, false, false> ARGS; \
    if (v.nobase) return v.uni ? FN<V, false, 3, false, false, true> ARGS : FN<V, false, 3, false, false, false> ARGS; \
    return v.uni ? FN<V, false, 0, false, false, true> ARGS : FN<V, false, 0, false, false, false> ARGS;

#define PS_PICK_OCC(FN, ARGS)                                                                          \
    if (MOVES || v.derived) {                                                                         \
        if (!MOVES && v.gstate && v.nobase) return v.uni ? FN<V, MOVES, 4, true, true> ARGS : FN<V, MOVES, 4, true, false> ARGS; \
        if (v.gstate && v.wmask) return v.uni ? FN<V, MOVES, 2, true, true> ARGS : FN<V, MOVES, 2, true, false> ARGS; \
        if (v.gstate) return v.uni ? FN<V, MOVES, 1, true, true> ARGS : FN<V, MOVES, 1, true, false> ARGS; \
        if (!MOVES && v.nobase) return v.uni ? FN<V, MOVES, 3, true, true> ARGS : FN<V, MOVES, 3, true, false> ARGS; \
        return v.uni ? FN<V, MOVES, 0, true, true> ARGS : FN<V, MOVES, 0, true, false> ARGS; \
    }                                                                                                 \
    if (v.gstate && v.nobase) return v.uni ? FN<V, false, 4, false, true> ARGS : FN<V, false, 4, false, false> ARGS; \
    if (v.gstate) return v.uni ? FN<V, false, 1, false, true> ARGS : FN<V, false, 1, false, false> ARGS; \
    if (v.nobase) return v.uni ? FN<V, false, 3, false, true> ARGS : FN<V, false, 3, false, false> ARGS; \
    return v.uni ? FN<V, false, 0, false, true> ARGS : FN<V, false, 0, false, false> ARGS;

template <typename V, bool MOVES>
cudaError_t eval_launch(Variant v, const EvalParams &p, LaunchCfg cfg, cudaStream_t s) {
    PS_PICK(launch_one, (p, cfg, s))
}

template <typename V, bool MOVES>
cudaError_t eval_occupancy(Variant v, int block, size_t smem, int *n) {
    PS_PICK_OCC(occ_one, (block, smem, n))
}

}  // namespace ps
