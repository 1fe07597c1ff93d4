// ps_launch.h — host-side launch interface of the evaluator variants.
#pragma once
#include <cuda_runtime.h>
#include "ps_eval.cuh"

namespace ps {

struct LaunchCfg {
    int grid, block;
    size_t smem;
};

struct Variant {
    bool gstate;    // per-candidate state in global memory
    bool record;    // base recording (checkpoints)
    bool derived;   // greedy channel mode
    bool uni;       // microbatch-symmetric instance tables
    bool wmask;     // (global state) nonzero-word masks over the pending-transfer sets
    bool nobase;    // (materialised, shared-memory state) no recorded base: the full-simulation build
};

// One translation unit per (ledger value type V, move-encoded candidates).
template <typename V, bool MOVES>
cudaError_t eval_launch(Variant v, const EvalParams &p, LaunchCfg cfg, cudaStream_t stream);
template <typename V, bool MOVES>
cudaError_t eval_occupancy(Variant v, int block, size_t smem, int *blocks_per_sm);

}  // namespace ps
