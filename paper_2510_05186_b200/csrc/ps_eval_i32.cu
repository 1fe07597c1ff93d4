// Evaluator variants with a 32-bit memory ledger (byte quantities fit after gcd scaling).
#include "ps_eval_impl.cuh"
namespace ps {
template cudaError_t eval_launch<int>(bool, bool, bool, const EvalParams &, LaunchCfg, cudaStream_t);
template cudaError_t eval_occupancy<int>(bool, bool, int, size_t, int *);
}
