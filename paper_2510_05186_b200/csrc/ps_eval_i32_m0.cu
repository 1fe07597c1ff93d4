// Evaluator variants: ledger value type int, move-encoded candidates = false.
#include "ps_eval_impl.cuh"
namespace ps {
template cudaError_t eval_launch<int, false>(Variant, const EvalParams &, LaunchCfg, cudaStream_t);
template cudaError_t eval_occupancy<int, false>(Variant, int, size_t, int *);
}
