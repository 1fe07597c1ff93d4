// Evaluator variants: ledger value type int, move-encoded candidates = true.
#include "ps_eval_impl.cuh"
namespace ps {
template cudaError_t eval_launch<int, true>(Variant, const EvalParams &, LaunchCfg, cudaStream_t);
template cudaError_t eval_occupancy<int, true>(Variant, int, size_t, int *);
}
