// Evaluator variants: ledger value type long long, move-encoded candidates = true.
#include "ps_eval_impl.cuh"
namespace ps {
template cudaError_t eval_launch<long long, true>(Variant, const EvalParams &, LaunchCfg, cudaStream_t);
template cudaError_t eval_occupancy<long long, true>(Variant, int, size_t, int *);
}
