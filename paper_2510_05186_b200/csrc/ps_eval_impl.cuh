// ps_eval_impl.cuh — instantiation helpers for ps_launch.h (included once per ledger width).
#pragma once
#include "ps_launch.h"

namespace ps {

template <typename V, bool MOVES, bool GSTATE, bool REC>
static cudaError_t launch_one(const EvalParams &p, LaunchCfg cfg, cudaStream_t stream) {
    auto fn = eval_kernel<V, MOVES, GSTATE, REC>;
    cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)cfg.smem);
    if (e != cudaSuccess) return e;
    fn<<<cfg.grid, cfg.block, cfg.smem, stream>>>(p);
    return cudaGetLastError();
}

template <typename V, bool MOVES, bool GSTATE>
static cudaError_t occ_one(int block, size_t smem, int *n) {
    auto fn = eval_kernel<V, MOVES, GSTATE, false>;
    cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    return cudaOccupancyMaxActiveBlocksPerMultiprocessor(n, fn, block, smem);
}

template <typename V>
cudaError_t eval_launch(bool moves, bool gstate, bool record, const EvalParams &p, LaunchCfg cfg, cudaStream_t s) {
    if (record) return launch_one<V, false, false, true>(p, cfg, s);
    if (moves) return gstate ? launch_one<V, true, true, false>(p, cfg, s) : launch_one<V, true, false, false>(p, cfg, s);
    return gstate ? launch_one<V, false, true, false>(p, cfg, s) : launch_one<V, false, false, false>(p, cfg, s);
}

template <typename V>
cudaError_t eval_occupancy(bool moves, bool gstate, int block, size_t smem, int *n) {
    if (moves) return gstate ? occ_one<V, true, true>(block, smem, n) : occ_one<V, true, false>(block, smem, n);
    return gstate ? occ_one<V, false, true>(block, smem, n) : occ_one<V, false, false>(block, smem, n);
}

}  // namespace ps
