// ps_launch.h — host-side launch interface of the evaluator variants (one TU per ledger width).
#pragma once
#include <cuda_runtime.h>
#include "ps_eval.cuh"

namespace ps {

struct LaunchCfg {
    int grid, block;
    size_t smem;
};

// Variant = (ledger value type V, move-encoded candidates, state in global memory, base recording).
template <typename V>
cudaError_t eval_launch(bool moves, bool gstate, bool record, const EvalParams &p, LaunchCfg cfg,
                        cudaStream_t stream);
template <typename V>
cudaError_t eval_occupancy(bool moves, bool gstate, int block, size_t smem, int *blocks_per_sm);

}  // namespace ps
