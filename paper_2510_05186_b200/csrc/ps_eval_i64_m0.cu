// Evaluator variants: ledger value type long long, move-encoded candidates = false.
#include "ps_eval_impl.cuh"
namespace ps {
template cudaError_t eval_launch<long long, false>(Variant, const EvalParams &, LaunchCfg, cudaStream_t);
template cudaError_t eval_occupancy<long long, false>(Variant, int, size_t, int *);
}
