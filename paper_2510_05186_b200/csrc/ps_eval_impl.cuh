// ps_eval_impl.cuh — instantiation helpers for ps_launch.h (included once per SEG TU).
#pragma once
#include "ps_launch.h"

namespace ps {

template <int SEG, typename V, bool MOVES, bool GSTATE>
static cudaError_t launch_one(const EvalParams &p, LaunchCfg cfg, cudaStream_t stream) {
    auto fn = eval_kernel<SEG, V, MOVES, GSTATE>;
    cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)cfg.smem);
    if (e != cudaSuccess) return e;
    fn<<<cfg.grid, cfg.block, cfg.smem, stream>>>(p);
    return cudaGetLastError();
}

template <int SEG, typename V, bool MOVES, bool GSTATE>
static cudaError_t occ_one(int block, size_t smem, int *n) {
    auto fn = eval_kernel<SEG, V, MOVES, GSTATE>;
    cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    return cudaOccupancyMaxActiveBlocksPerMultiprocessor(n, fn, block, smem);
}

#define PS_DISPATCH(FN, ...)                                                                        \
    if (v64) {                                                                                      \
        if (moves) return gstate ? FN<SEG, long long, true, true>(__VA_ARGS__)                     \
                                 : FN<SEG, long long, true, false>(__VA_ARGS__);                   \
        return gstate ? FN<SEG, long long, false, true>(__VA_ARGS__)                               \
                      : FN<SEG, long long, false, false>(__VA_ARGS__);                             \
    }                                                                                               \
    if (moves) return gstate ? FN<SEG, int, true, true>(__VA_ARGS__) : FN<SEG, int, true, false>(__VA_ARGS__); \
    return gstate ? FN<SEG, int, false, true>(__VA_ARGS__) : FN<SEG, int, false, false>(__VA_ARGS__);

template <int SEG>
cudaError_t eval_launch(bool v64, bool moves, bool gstate, const EvalParams &p, LaunchCfg cfg,
                        cudaStream_t stream) {
    PS_DISPATCH(launch_one, p, cfg, stream)
}

template <int SEG>
cudaError_t eval_occupancy(bool v64, bool moves, bool gstate, int block, size_t smem, int *n) {
    PS_DISPATCH(occ_one, block, smem, n)
}

#define PS_INSTANTIATE(SEG)                                                                          \
    template cudaError_t eval_launch<SEG>(bool, bool, bool, const EvalParams &, LaunchCfg, cudaStream_t); \
    template cudaError_t eval_occupancy<SEG>(bool, bool, bool, int, size_t, int *);

}  // namespace ps
