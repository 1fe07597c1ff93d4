// ps_launch.h — host-side launch interface of the evaluator variants (one TU per SEG).
#pragma once
#include <cuda_runtime.h>
#include "ps_eval.cuh"

namespace ps {

struct LaunchCfg {
    int grid, block;
    size_t smem;
};

// Variant = (SEG, 64-bit ledger values, move-encoded candidates, state in global memory).
template <int SEG>
cudaError_t eval_launch(bool v64, bool moves, bool gstate, const EvalParams &p, LaunchCfg cfg,
                        cudaStream_t stream);
template <int SEG>
cudaError_t eval_occupancy(bool v64, bool moves, bool gstate, int block, size_t smem, int *blocks_per_sm);

}  // namespace ps
