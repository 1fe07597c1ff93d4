// Evaluator variants with a 64-bit memory ledger.
#include "ps_eval_impl.cuh"
namespace ps {
template cudaError_t eval_launch<long long>(bool, bool, bool, const EvalParams &, LaunchCfg, cudaStream_t);
template cudaError_t eval_occupancy<long long>(bool, bool, int, size_t, int *);
}
